// l2f_device.cuh -- device-side building blocks of the batched quadrotor env step
// (arXiv 2311.13081).  One env per thread; every function here operates on registers.
// Shared by the single-step kernel, the open-loop rollout and the tcgen05 MLP rollout so
// that T x l2f_step and l2f_rollout(T) execute the same arithmetic.
//
// Citations: P:n = /root/reference/PAPER.md line n; Qn = DESIGN.md section 3 readings.
// This file is independent of oracle/ (no shared code, tables or constants).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Debug build (-DL2F_DEBUG_CHECKS, scripts/debug_checks.sh): bounds and protocol checks on every
// global / shared / tensor-memory index the kernels form, and bounded mbarrier waits; a failed
// check prints and traps.  (compute-sanitizer is not available on the measurement pool.)
#ifdef L2F_DEBUG_CHECKS
#define L2F_CHECK(cond, what)                                                                          \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("L2F_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,      \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define L2F_CHECK(cond, what) \
    do {                      \
    } while (0)
#endif

namespace l2f {

constexpr int kStateDim = 17;
constexpr int kObsCore = 18;
constexpr int kMaxHist = 32;
constexpr int kMaxStages = 8;
constexpr int kStatsLen = 8;
constexpr int kTraceFields = 32;
constexpr int kResetScratch = 40;  // uint4 per warp for reset_env_warp

enum : uint32_t {
    F_OBS_NOISE = 1u << 0,
    F_ACTION_NOISE = 1u << 1,
    F_TERMINATION = 1u << 2,
    F_AUTO_RESET = 1u << 3,
    F_DISTURBANCE = 1u << 4,
    F_DOMAIN_RAND = 1u << 5,
    F_NO_ROTOR_DELAY = 1u << 6,  // ablation (Table II "Rotor Delay"): w_m set to the setpoint
};
enum : uint32_t { D_TERM = 1, D_TRUNC = 2, D_DIV = 4, D_RESET = 8 };
enum : uint32_t { S_ACT = 1, S_OBS = 2, S_RESET = 3, S_DIST = 4, S_DR = 5, S_RAND_ACT = 6 };

// Reward weights + exploration sigma of one curriculum stage, fp32.
struct StageW {
    float C_rp, C_rq, C_rv, C_rw, C_ra, C_rab[4], C_rs, sigma_a;
};

// Launch-uniform parameters, passed by value (constant bank) to every kernel.
struct DevParams {
    uint32_t key0, key1;       // Philox key = seed (Q20)
    uint32_t rk0[10], rk1[10]; // Philox4x32-10 round keys (key + r * Weyl constants)
    uint32_t flags;
    int32_t n_hist;
    int32_t hist_slot0;        // t0 mod N_H (0 when N_H = 0)
    int32_t max_ep;
    uint32_t id_offset;        // global env id of local env 0
    int64_t n;                 // envs
    uint32_t t0;               // step counter at launch
    // integration
    float dt, half_dt, dt_6, dt2_6;
    // RK4 of the linear rotor lag (rk4_step): stage values u + d beta_j, result u + d R
    float m_beta2, m_beta3, m_beta4, m_R;
    // nominal parameters; DR factors scale mass, J, thrust coefficients (Q19)
    float mass, J[3], c[3], ctau, inv_tm, rpm_min, rpm_max, gravity, rpm_half_span, inv_rpm_span2;
    float rx[4], ry[4], spin[4];
    float2 rxy[4];                 // (ry_i, -rx_i): roll/pitch torque arms per rotor, packed
    float inv_mass, iJ[3], dJ[3];  // nominal 1/m, 1/J_ii, (Jz-Jy, Jx-Jz, Jy-Jx): DR-free fast path
    // reset distribution (Q17-Q19)
    float init_pos, init_angle, init_vel, init_angvel, init_rpm_lo, init_rpm_hi;
    float dist_force, dist_torque, dr_lo, dr_hi;
    // reset sampling table: value (Philox slot b, component c) = rs_lo + rs_span * u (host-built
    // from the ranges above with the span rounded in fp32; reset_values)
    float4 rs_lo[8], rs_span[8];
    // observation noise (Q8), termination (Q14)
    float obs_sigma[4];
    float term_pos, term_vel2, term_angvel2;
    // curriculum slice covering [t0, t0 + T): stage[j] holds the weights of steps
    // [stage_end[j-1], stage_end[j]); host-computed, so the kernel only compares step indices
    int32_t n_stages;
    uint32_t stage_end[kMaxStages];
    StageW stage[kMaxStages];
};

// Feature flags of a launch: the run-time P.flags, or a compile-time set kF for kernels
// specialised on one feature mix (kAnyFlags = read P.flags), so flag tests fold away.
constexpr uint32_t kAnyFlags = 0xFFFFFFFFu;
template <uint32_t kF>
__device__ __forceinline__ uint32_t flags_of(const DevParams& P)
{
    return kF == kAnyFlags ? P.flags : kF;
}

// Workspace views: structure of arrays of float4 groups plus a tail (grp_load): a warp moves each
// group as 512 contiguous bytes with one 128-bit access per thread, and no byte is padding.
struct DevBufs {
    float4* state;     // [4][N] float4 (p, q, v, w, w_m0..2) + [N] float (w_m3)
    float4* dist;      // [1][N] float4 (f_r, tau_x) + [N] float2 (tau_y, tau_z)
    float4* dr;        // [1][N] float4 (m, J_xx, J_yy, J_zz) + [N] float (thrust scale)
    float4* hist;      // [N_H][N] ring: slot (tau mod N_H) = action applied at step tau
    int32_t* hist_t0;  // [N] first step of the current episode: ring entries with tau < hist_t0
    float4* hist_fill; // [N]   read as hist_fill (the episode's initial history, Q10)
    int32_t* ep_step;  // [N]
    float* ep_return;  // [N]
    double* slots;     // [n_slots][8] per-block statistics partials
    int32_t n_slots;
};

// Registers of one env.
struct EnvReg {
    float s[kStateDim];
    float dist[6];
    float dr[5];
    int32_t ep_step;
    float ep_return;
};

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (Random123), counter = (env id, t, stream, block), key = seed (Q20).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ k0;
        c2 = hi0 ^ c3 ^ k1;
        c1 = lo1;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// Same rounds with the 10 round keys precomputed on the host (DevParams.rk): the key
// schedule is launch-uniform, so each round is 2 IMAD.WIDE + 2 LOP3 with constant-bank keys.
__device__ __forceinline__ uint4 philox_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           const uint32_t (&rk0)[10], const uint32_t (&rk1)[10])
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ rk0[r];
        c2 = hi0 ^ c3 ^ rk1[r];
        c1 = lo1;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint4 draw(const DevParams& P, uint32_t gid, uint32_t t,
                                      uint32_t stream, uint32_t block)
{
    return philox_rk(gid, t, stream, block, P.rk0, P.rk1);
}

// u = (2 (x >> 9) + 1) 2^-24 = ((x >> 9) + 1/2) 2^-23, exact in fp32 (Q20).  Built from the
// bits: 1 + (x >> 9) 2^-23 is the float with exponent 0 and mantissa x >> 9; subtracting
// 1 - 2^-24 is exact (Sterbenz), so no int->float conversion is needed.
__device__ __forceinline__ float unif(uint32_t x)
{
    return __uint_as_float(0x3F800000u | (x >> 9)) - 0.99999994039535522f;
}

// ln(u) for u in (0,1): log1p series near 1 (where MUFU.LG2's absolute error would swamp
// the tiny result), MUFU.LG2 elsewhere (relative error <= ~3e-6 there).
__device__ __forceinline__ float ln_unit(float u)
{
    const float x = u - 1.0f;  // exact for u >= 1/2
    float p = fmaf(x, -1.0f / 6.0f, 0.2f);
    p = fmaf(x, p, -0.25f);
    p = fmaf(x, p, 1.0f / 3.0f);
    p = fmaf(x, p, -0.5f);
    p = fmaf(x, p, 1.0f);
    const float series = x * p;
    const float l = __log2f(u) * 0.69314718055994531f;
    return (x > -0.0625f) ? series : l;
}

// Box-Muller (Q20): r = sqrt(-2 ln u1), theta = 2 pi u2.
__device__ __forceinline__ void box_muller(uint32_t xa, uint32_t xb, float& z0, float& z1)
{
    const float u1 = unif(xa), u2 = unif(xb);
    const float y = -2.0f * ln_unit(u1);
    const float r = y * rsqrtf(y);
    float sn, cs;
    __sincosf(6.28318530717958648f * u2, &sn, &cs);
    z0 = r * cs;
    z1 = r * sn;
}

// Both Box-Muller pairs of one Philox block, (x.x, x.y) -> z0, z1 and (x.z, x.w) -> z2, z3, in
// packed f32x2 arithmetic (FADD2 / FFMA2 / FMUL2): every element goes through the same
// round-to-nearest operations as box_muller, so the results are identical to two calls.
__device__ __forceinline__ void box_muller2(uint4 x, float z[4])
{
    const float c = -0.99999994039535522f;
    const float2 u1 = __fadd2_rn(make_float2(__uint_as_float(0x3F800000u | (x.x >> 9)),
                                             __uint_as_float(0x3F800000u | (x.z >> 9))), make_float2(c, c));
    const float2 u2 = __fadd2_rn(make_float2(__uint_as_float(0x3F800000u | (x.y >> 9)),
                                             __uint_as_float(0x3F800000u | (x.w >> 9))), make_float2(c, c));
    const float2 xm = __fadd2_rn(u1, make_float2(-1.0f, -1.0f));
    float2 p = __ffma2_rn(xm, make_float2(-1.0f / 6.0f, -1.0f / 6.0f), make_float2(0.2f, 0.2f));
    p = __ffma2_rn(xm, p, make_float2(-0.25f, -0.25f));
    p = __ffma2_rn(xm, p, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
    p = __ffma2_rn(xm, p, make_float2(-0.5f, -0.5f));
    p = __ffma2_rn(xm, p, make_float2(1.0f, 1.0f));
    const float2 series = __fmul2_rn(xm, p);
    const float2 lg = __fmul2_rn(make_float2(__log2f(u1.x), __log2f(u1.y)),
                                 make_float2(0.69314718055994531f, 0.69314718055994531f));
    const float2 ln = make_float2(xm.x > -0.0625f ? series.x : lg.x, xm.y > -0.0625f ? series.y : lg.y);
    const float2 y = __fmul2_rn(make_float2(-2.0f, -2.0f), ln);
    const float2 r = __fmul2_rn(y, make_float2(rsqrtf(y.x), rsqrtf(y.y)));
    const float2 th = __fmul2_rn(make_float2(6.28318530717958648f, 6.28318530717958648f), u2);
    float s0, c0, s1, c1;
    __sincosf(th.x, &s0, &c0);
    __sincosf(th.y, &s1, &c1);
    const float2 za = __fmul2_rn(make_float2(r.x, r.x), make_float2(c0, s0));
    const float2 zb = __fmul2_rn(make_float2(r.y, r.y), make_float2(c1, s1));
    z[0] = za.x;
    z[1] = za.y;
    z[2] = zb.x;
    z[3] = zb.y;
}

__device__ __forceinline__ const StageW& stage_of(const DevParams& P, uint32_t t)
{
    int k = 0;
    for (int j = 0; j + 1 < P.n_stages; ++j) k += (t >= P.stage_end[j]) ? 1 : 0;
    return P.stage[k];
}

// Last step (exclusive) of launch stage sg when the launch covers [t0, t0 + T).
__device__ __forceinline__ uint32_t stage_stop(const DevParams& P, int sg, uint32_t t_last)
{
    return (sg + 1 < P.n_stages) ? min(P.stage_end[sg], t_last) : t_last;
}

// ---------------------------------------------------------------------------------------
// Dynamics: per-step constants of one env, then f(s).
// ---------------------------------------------------------------------------------------
struct Phys {
    float c0, c1, c2;       // thrust coefficients x DR thrust scale
    float inv_m;
    float Jx, Jy, Jz, iJx, iJy, iJz;
    float dJzy, dJxz, dJyx; // Jz - Jy, Jx - Jz, Jy - Jx (gyroscopic term)
};

template <bool kDR>
__device__ __forceinline__ void make_phys(const DevParams& P, const EnvReg& e, Phys& ph)
{
    if constexpr (kDR) {
        ph.c0 = P.c[0] * e.dr[4];
        ph.c1 = P.c[1] * e.dr[4];
        ph.c2 = P.c[2] * e.dr[4];
        ph.inv_m = __fdividef(1.0f, P.mass * e.dr[0]);
        ph.Jx = P.J[0] * e.dr[1];
        ph.Jy = P.J[1] * e.dr[2];
        ph.Jz = P.J[2] * e.dr[3];
        ph.dJzy = ph.Jz - ph.Jy;
        ph.dJxz = ph.Jx - ph.Jz;
        ph.dJyx = ph.Jy - ph.Jx;
        ph.iJx = __fdividef(1.0f, ph.Jx);
        ph.iJy = __fdividef(1.0f, ph.Jy);
        ph.iJz = __fdividef(1.0f, ph.Jz);
    } else {  // launch-uniform constants (constant-bank operands, no registers)
        ph.c0 = P.c[0];
        ph.c1 = P.c[1];
        ph.c2 = P.c[2];
        ph.inv_m = P.inv_mass;
        ph.Jx = P.J[0];
        ph.Jy = P.J[1];
        ph.Jz = P.J[2];
        ph.dJzy = P.dJ[0];
        ph.dJxz = P.dJ[1];
        ph.dJyx = P.dJ[2];
        ph.iJx = P.iJ[0];
        ph.iJy = P.iJ[1];
        ph.iJz = P.iJ[2];
    }
}

// Derivative of the coupled part y = (q, w) of the state, given the rotor speeds m of the RK4
// stage: q' = 1/2 q (x) (0,w); w' = J^-1 (tau - w x J w); plus the
// linear acceleration av = v' = (R e_z T + f_r)/m - g e_z, which feeds nothing back.
// y = (qw, qx, qy, qz, wx, wy, wz).
constexpr int kY = 7;
__device__ __forceinline__ void deriv(const DevParams& P, const Phys& ph, const float* d, const float* y,
                                      float2 mA, float2 mB, float* dy, float av[3])
{
    // rotor thrusts packed as (f0, f2) and (f1, f3) from the rotor speeds (m0, m2), (m1, m3)
    const float2 c2 = make_float2(ph.c2, ph.c2), c1 = make_float2(ph.c1, ph.c1), c0 = make_float2(ph.c0, ph.c0);
    const float2 fA = __ffma2_rn(__ffma2_rn(c2, mA, c1), mA, c0);
    const float2 fB = __ffma2_rn(__ffma2_rn(c2, mB, c1), mB, c0);
    const float2 sp = __fadd2_rn(fA, fB);  // (f0 + f1, f2 + f3)
    const float T = sp.x + sp.y;
    // (tau_x, tau_y) = (d3, d4) + sum_i (ry_i, -rx_i) f_i, rotor order 0..3 as in the scalar sum
    float2 txy = make_float2(d[3], d[4]);
    txy = __ffma2_rn(P.rxy[0], make_float2(fA.x, fA.x), txy);
    txy = __ffma2_rn(P.rxy[1], make_float2(fB.x, fB.x), txy);
    txy = __ffma2_rn(P.rxy[2], make_float2(fA.y, fA.y), txy);
    txy = __ffma2_rn(P.rxy[3], make_float2(fB.y, fB.y), txy);
    float tz = fmaf(P.spin[0], fA.x, 0.0f);
    tz = fmaf(P.spin[1], fB.x, tz);
    tz = fmaf(P.spin[2], fA.y, tz);
    tz = fmaf(P.spin[3], fB.y, tz);
    tz = fmaf(P.ctau, tz, d[5]);
    const float qw = y[0], qx = y[1], qy = y[2], qz = y[3];
    const float wx = y[4], wy = y[5], wz = y[6];
    const float hx = 0.5f * wx, hy = 0.5f * wy, hz = 0.5f * wz;
    dy[0] = -(qx * hx + qy * hy + qz * hz);
    dy[1] = qw * hx + qy * hz - qz * hy;
    dy[2] = qw * hy - qx * hz + qz * hx;
    dy[3] = qw * hz + qx * hy - qy * hx;
    // third column of R(q): body z-axis in world
    const float r02 = 2.0f * (qx * qz + qw * qy);
    const float r12 = 2.0f * (qy * qz - qw * qx);
    const float r22 = 1.0f - 2.0f * (qx * qx + qy * qy);
    const float2 a01 = __fmul2_rn(__ffma2_rn(make_float2(r02, r12), make_float2(T, T), make_float2(d[0], d[1])),
                                  make_float2(ph.inv_m, ph.inv_m));
    av[0] = a01.x;
    av[1] = a01.y;
    av[2] = fmaf(fmaf(r22, T, d[2]), ph.inv_m, -P.gravity);
    // Euler: J w' = tau - w x (J w)
    const float cx = ph.dJzy * (wy * wz);
    const float cy = ph.dJxz * (wz * wx);
    const float cz = ph.dJyx * (wx * wy);
    dy[4] = (txy.x - cx) * ph.iJx;
    dy[5] = (txy.y - cy) * ph.iJy;
    dy[6] = (tz - cz) * ph.iJz;
}

// Float4-group SoA (DevBufs): components 0 .. 4 floor(C/4) - 1 of env i as float4 groups
// (element (c/4) N + i, lane c % 4), the C % 4 tail components as one float / float2 element
// i of an [N] array right after the groups.  Exact bytes (no padding), one 128-bit access per
// group and one 32/64-bit access for the tail.
template <int C>
__device__ __forceinline__ void grp_load(const float4* base, int64_t i, int64_t N, float* out)
{
    constexpr int G = C / 4, R = C % 4;
    L2F_CHECK(i >= 0 && i < N, "grp_load index");
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float4 v = base[g * N + i];
        out[4 * g] = v.x, out[4 * g + 1] = v.y, out[4 * g + 2] = v.z, out[4 * g + 3] = v.w;
    }
    if constexpr (R == 1) {
        out[4 * G] = reinterpret_cast<const float*>(base + G * N)[i];
    } else if constexpr (R == 2) {
        const float2 v = reinterpret_cast<const float2*>(base + G * N)[i];
        out[4 * G] = v.x, out[4 * G + 1] = v.y;
    }
    static_assert(R < 3, "tail of 0, 1 or 2 components");
}
// Scalar-access variant of grp_load (same layout): for kernels that read a state once, where
// 128-bit register quads only constrain the allocator of the hot loop that follows.
template <int C>
__device__ __forceinline__ void grp_load_scalar(const float4* base4, int64_t i, int64_t N, float* out)
{
    constexpr int G = C / 4, R = C % 4;
    L2F_CHECK(i >= 0 && i < N, "grp_load_scalar index");
    const float* base = reinterpret_cast<const float*>(base4);
#pragma unroll
    for (int c = 0; c < 4 * G; ++c) out[c] = base[((c / 4) * N + i) * 4 + (c % 4)];
#pragma unroll
    for (int c = 0; c < R; ++c) out[4 * G + c] = base[4 * G * N + i * R + c];
}

template <int C>
__device__ __forceinline__ void grp_store(float4* base, int64_t i, int64_t N, const float* v)
{
    constexpr int G = C / 4, R = C % 4;
    L2F_CHECK(i >= 0 && i < N, "grp_store index");
#pragma unroll
    for (int g = 0; g < G; ++g) base[g * N + i] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    if constexpr (R == 1) {
        reinterpret_cast<float*>(base + G * N)[i] = v[4 * G];
    } else if constexpr (R == 2) {
        reinterpret_cast<float2*>(base + G * N)[i] = make_float2(v[4 * G], v[4 * G + 1]);
    }
}

// SoA walkers: rows c = 0..C-1 of column i of a [C][N] array, visited in order with one
// 32-bit-stride IMAD.WIDE per access (the indexed form c * N + i with a 64-bit N costs two to
// three integer instructions per access).  N < 2^32.
template <int C, class T>
__device__ __forceinline__ void soa_load(const T* base, int64_t i, uint32_t n, T* out)
{
    L2F_CHECK(i >= 0 && i < (int64_t)n, "soa index");
    const T* q = base + i;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        out[c] = *q;
        q += n;
    }
}
template <int C, class T>
__device__ __forceinline__ void soa_load_ro(const T* __restrict__ base, int64_t i, uint32_t n, T* out)
{
    L2F_CHECK(i >= 0 && i < (int64_t)n, "soa index");
    const T* q = base + i;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        out[c] = __ldg(q);
        q += n;
    }
}
template <int C, class T>
__device__ __forceinline__ void soa_store(T* base, int64_t i, uint32_t n, const T* v)
{
    L2F_CHECK(i >= 0 && i < (int64_t)n, "soa index");
    T* q = base + i;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        *q = v[c];
        q += n;
    }
}

// Any NaN/Inf component makes the sum non-finite (a finite overflow to inf also counts:
// |x| > 1e38 is divergence in any sense).  Checked on the projected state s'.
__device__ __forceinline__ bool state_finite(const float* s)
{
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < kStateDim; ++i) sum += s[i];
    return isfinite(sum);
}

// The same decision for a state just produced by rk4_step from a step's inputs, from p, q, w
// alone: a non-finite v or w_m (or f_r, tau_r, action) cannot leave p' = p + h v + h^2/6 (a1 +
// a2 + a3), q' and w' all finite -- v enters p' directly, and w_m (before its clamp, which would
// map NaN to a bound) enters every stage's thrust, hence v' and w' (non-finite or overflowing).
__device__ __forceinline__ bool stepped_state_finite(const float* s)
{
    const float sum = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[10])) + (s[11] + s[12]);
    return isfinite(sum);
}

// out = a * h + b over the 7 coupled components: 3 packed FFMA2 pairs + 1 scalar FFMA.
__device__ __forceinline__ void pair_fma(const float* a, float h, const float* b, float* out)
{
    const float2 hh = make_float2(h, h);
#pragma unroll
    for (int i = 0; i + 1 < kY; i += 2) {
        const float2 r = __ffma2_rn(make_float2(a[i], a[i + 1]), hh, make_float2(b[i], b[i + 1]));
        out[i] = r.x;
        out[i + 1] = r.y;
    }
    out[kY - 1] = fmaf(a[kY - 1], h, b[kY - 1]);
}

// Classical RK4 at dt with zero-order-hold setpoints u (Q1), then q renormalisation and
// rotor-speed clamp (Q5).  Returns true if the result is non-finite.  The RK4 is
// evaluated in the algebraically identical form that exploits the structure of the ODE
// (DESIGN.md section 5.6), so only the coupled part y = (q, w) carries stage vectors:
//  * rotors: w_m' = (u - w_m)/T_m is linear with a constant input, so with d = w_m0 - u the
//    RK4 stage values are u + d beta_j and the RK4 result is u + d R (R = the RK4 stability
//    polynomial at -dt/T_m; beta_j, R precomputed in FP64 on the host);
//  * velocity: v' = a(q, w_m) does not depend on v, so v_new = v + h/6 (a1 + 2 a2 + 2 a3 + a4)
//    needs no stage velocities;
//  * position: p' = v with stage velocities v, v + h/2 a1, v + h/2 a2, v + h a3 gives
//    p_new = p + h v + h^2/6 (a1 + a2 + a3).
__device__ __forceinline__ bool rk4_step(const DevParams& P, const Phys& ph, const float* d, const float u[4],
                                         float* s)
{
    float y0[kY] = {s[3], s[4], s[5], s[6], s[10], s[11], s[12]};
    // rotors packed as (0, 2) and (1, 3): d = w_m0 - u, stage speeds u + d beta_j
    const float2 uA = make_float2(u[0], u[2]), uB = make_float2(u[1], u[3]);
    const float2 dA = make_float2(s[13] - u[0], s[15] - u[2]), dB = make_float2(s[14] - u[1], s[16] - u[3]);
    float acc[kY], tmp[kY], k[kY], a[3], asum[3], vacc[3];
    deriv(P, ph, d, y0, make_float2(s[13], s[15]), make_float2(s[14], s[16]), k, a);
#pragma unroll
    for (int i = 0; i < 3; ++i) asum[i] = vacc[i] = a[i];
#pragma unroll
    for (int i = 0; i < kY; ++i) acc[i] = k[i];
    pair_fma(k, P.half_dt, y0, tmp);
    float2 b = make_float2(P.m_beta2, P.m_beta2);
    deriv(P, ph, d, tmp, __ffma2_rn(dA, b, uA), __ffma2_rn(dB, b, uB), k, a);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        asum[i] += a[i];
        vacc[i] = fmaf(a[i], 2.0f, vacc[i]);
    }
    pair_fma(k, 2.0f, acc, acc);
    pair_fma(k, P.half_dt, y0, tmp);
    b = make_float2(P.m_beta3, P.m_beta3);
    deriv(P, ph, d, tmp, __ffma2_rn(dA, b, uA), __ffma2_rn(dB, b, uB), k, a);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        asum[i] += a[i];
        vacc[i] = fmaf(a[i], 2.0f, vacc[i]);
    }
    pair_fma(k, 2.0f, acc, acc);
    pair_fma(k, P.dt, y0, tmp);
    b = make_float2(P.m_beta4, P.m_beta4);
    deriv(P, ph, d, tmp, __ffma2_rn(dA, b, uA), __ffma2_rn(dB, b, uB), k, a);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        s[i] = fmaf(P.dt2_6, asum[i], fmaf(P.dt, s[7 + i], s[i]));  // position (pre-step v)
        s[7 + i] = fmaf(P.dt_6, vacc[i] + a[i], s[7 + i]);
    }
    {
        const float2 h6 = make_float2(P.dt_6, P.dt_6);
#pragma unroll
        for (int i = 0; i + 1 < kY; i += 2) {
            const float2 sm = __fadd2_rn(make_float2(acc[i], acc[i + 1]), make_float2(k[i], k[i + 1]));
            const float2 r = __ffma2_rn(h6, sm, make_float2(y0[i], y0[i + 1]));
            y0[i] = r.x;
            y0[i + 1] = r.y;
        }
        y0[kY - 1] = fmaf(P.dt_6, acc[kY - 1] + k[kY - 1], y0[kY - 1]);
    }
    const float2 R = make_float2(P.m_R, P.m_R);
    const float2 wA = __ffma2_rn(dA, R, uA), wB = __ffma2_rn(dB, R, uB);
    s[13] = wA.x;
    s[14] = wB.x;
    s[15] = wA.y;
    s[16] = wB.y;
    const float n2 = (y0[0] * y0[0] + y0[1] * y0[1]) + (y0[2] * y0[2] + y0[3] * y0[3]);
    const float inv = rsqrtf(n2);
#pragma unroll
    for (int i = 0; i < 4; ++i) s[3 + i] = y0[i] * inv;
#pragma unroll
    for (int i = 0; i < 3; ++i) s[10 + i] = y0[4 + i];
#pragma unroll
    for (int i = 13; i < 17; ++i) s[i] = fminf(fmaxf(s[i], P.rpm_min), P.rpm_max);
    return !stepped_state_finite(s);
}

// ---------------------------------------------------------------------------------------
// Result of one transition (before any reset).
// ---------------------------------------------------------------------------------------
struct Trans {
    float a[4];      // applied action a'
    float reward;
    uint32_t flags;  // D_TERM | D_TRUNC | D_DIV
    int32_t len;     // episode length if it ended
    float ret;       // episode return if it ended
};

// One env transition s_t -> s_{t+1}: exploration noise + clip (Q7),
// action map, RK4 dynamics, reward on s' (Q12), termination (Q14),
// truncation (Q15).  Episode counters are advanced; the caller handles history and reset.
// Exploration-noise normals of step t (stream ACT, Q20); zeros when the feature is off.
template <uint32_t kF = kAnyFlags>
__device__ __forceinline__ void action_noise(const DevParams& P, uint32_t gid, uint32_t t, float z[4])
{
    z[0] = z[1] = z[2] = z[3] = 0.0f;
    if (flags_of<kF>(P) & F_ACTION_NOISE) {
        box_muller2(draw(P, gid, t, S_ACT, 0), z);
    }
}

// Reward r(s, a, s') on the post-transition state (Q12): the same function serves
// the step and the replay-buffer recalculation (l2f_recompute_rewards).
__device__ __forceinline__ float reward_of(const StageW& W, const float* s, const float a[4])
{
    const float pp = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
    const float vv = s[7] * s[7] + s[8] * s[8] + s[9] * s[9];
    const float ww = s[10] * s[10] + s[11] * s[11] + s[12] * s[12];
    float aa = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float d = a[i] - W.C_rab[i];
        aa = fmaf(d, d, aa);
    }
    float r = W.C_rs;
    r = fmaf(-W.C_rp, pp, r);
    r = fmaf(-W.C_rq, fmaf(-s[3], s[3], 1.0f), r);
    r = fmaf(-W.C_rv, vv, r);
    r = fmaf(-W.C_rw, ww, r);
    r = fmaf(-W.C_ra, aa, r);
    return r;
}

// Privileged critic observation o_c = {p, R, v, w, w_m, f_r, tau_r}, 28-D, noise-free
// (P:137-139).
constexpr int kObsCritic = 28;
__device__ __forceinline__ void observe_critic(const float* s, const float* dist, float o[kObsCritic])
{
    const float qw = s[3], qx = s[4], qy = s[5], qz = s[6];
    o[0] = s[0];
    o[1] = s[1];
    o[2] = s[2];
    // R(q) with every multiply-add written out as fmaf: the compiler's own contraction of
    // a*b +- c*d may pick either product, and differently in two builds of this function
    // (seen between the debug-check build's specialised and generic step kernels)
    const float x2 = qx + qx, y2 = qy + qy, z2 = qz + qz;  // exact doublings
    const float wx2 = qw * x2, wy2 = qw * y2, wz2 = qw * z2;
    o[3] = fmaf(-qy, y2, fmaf(-qz, z2, 1.0f));
    o[4] = fmaf(qx, y2, -wz2);
    o[5] = fmaf(qx, z2, wy2);
    o[6] = fmaf(qx, y2, wz2);
    o[7] = fmaf(-qx, x2, fmaf(-qz, z2, 1.0f));
    o[8] = fmaf(qy, z2, -wx2);
    o[9] = fmaf(qx, z2, -wy2);
    o[10] = fmaf(qy, z2, wx2);
    o[11] = fmaf(-qx, x2, fmaf(-qy, y2, 1.0f));
#pragma unroll
    for (int j = 0; j < 10; ++j) o[12 + j] = s[7 + j];  // v, w, w_m
#pragma unroll
    for (int j = 0; j < 6; ++j) o[22 + j] = dist[j];
}

// W: the curriculum stage of step t (stage_of), hoisted by the callers' stage loops.
// kDR: per-env domain-randomised parameters (compile-time so the DR-free path keeps the
// nominal parameters in the constant bank instead of registers).
template <bool kDR, uint32_t kF = kAnyFlags>
__device__ __forceinline__ void transition(const DevParams& P, const StageW& W, EnvReg& e, uint32_t gid,
                                           uint32_t t, const float a_in[4], const float z[4], Trans& o)
{
    const uint32_t flags = flags_of<kF>(P);
    // branch-free on the feature flags (selects), so several envs' transitions can share one
    // basic block and interleave their dependency chains
    const bool act_noise = (flags & F_ACTION_NOISE) != 0;
    const bool no_delay = (flags & F_NO_ROTOR_DELAY) != 0;
    float u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float v = act_noise ? fmaf(W.sigma_a, z[i], a_in[i]) : a_in[i];
        o.a[i] = fminf(fmaxf(v, -1.0f), 1.0f);
        u[i] = fmaf(o.a[i] + 1.0f, P.rpm_half_span, P.rpm_min);
        // ablation: rotors reach the setpoint instantly
        e.s[13 + i] = no_delay ? u[i] : e.s[13 + i];
    }
    Phys ph;
    make_phys<kDR>(P, e, ph);
    const bool div = rk4_step(P, ph, e.dist, u, e.s);

    const float* s = e.s;
    const float vv = s[7] * s[7] + s[8] * s[8] + s[9] * s[9];
    const float ww = s[10] * s[10] + s[11] * s[11] + s[12] * s[12];
    const float rw = reward_of(W, s, o.a);
    const float r = div ? 0.0f : rw;  // Q26
    const float pinf = fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2])));
    const bool out = (pinf > P.term_pos) | (vv > P.term_vel2) | (ww > P.term_angvel2);
    const bool term = div | (((flags & F_TERMINATION) != 0) & out);
    e.ep_step += 1;
    e.ep_return += r;
    const bool trunc = (!term) & (P.max_ep > 0) & (e.ep_step >= P.max_ep);
    o.reward = r;
    o.flags = (term ? D_TERM : 0u) | (trunc ? D_TRUNC : 0u) | (div ? D_DIV : 0u);
    o.len = e.ep_step;
    o.ret = e.ep_return;
}

__device__ __forceinline__ float uab(float a, float b, uint32_t x) { return fmaf(b - a, unif(x), a); }

// Philox blocks of one reset (Q20): RESET 0..3 at slots 0..3, DIST 0..1 at slots 4..5,
// DR 0..1 at slots 6..7.
__device__ __forceinline__ int reset_nblocks(const DevParams& P)
{
    return (P.flags & (F_DISTURBANCE | F_DOMAIN_RAND)) ? 8 : 4;
}

__device__ __forceinline__ uint4 reset_block(const DevParams& P, uint32_t gid, uint32_t ctr, int b)
{
    const uint32_t stream = b < 4 ? S_RESET : (b < 6 ? S_DIST : S_DR);
    const uint32_t blk = (uint32_t)(b < 4 ? b : (b < 6 ? b - 4 : b - 6));
    return draw(P, gid, ctr, stream, blk);
}

// The four sampled values of reset slot b (Q17-Q19): lo + span * u per uniform
// of the slot's Philox block.  Slot 0: p_x, p_y, p_z, axis cos-polar c_z; slot 1: axis azimuth
// phi, rotation angle theta, v_x, v_y; slot 2: v_z, w; slot 3: rotor speeds; slots 4-5:
// disturbance force, torque; slots 6-7: DR factors (m, J_xx, J_yy, J_zz, thrust scale).
__device__ __forceinline__ float4 reset_values(const DevParams& P, int b, uint4 x)
{
    const float4 lo = P.rs_lo[b], sp = P.rs_span[b];
    return make_float4(fmaf(sp.x, unif(x.x), lo.x), fmaf(sp.y, unif(x.y), lo.y), fmaf(sp.z, unif(x.z), lo.z),
                       fmaf(sp.w, unif(x.w), lo.w));
}

// The sampling table in shared memory (tab[b] = lo, tab[8 + b] = span of slot b): the
// cooperative reset reads slot (lane mod nb), and a lane-divergent constant-bank index
// serialises 8 ways.  Threads 0..15 copy; the caller synchronises before the first use.  (Kernels
// without a barrier to spare pass tab = nullptr and index the constant bank instead.)
__device__ __forceinline__ void reset_table_to_smem(const DevParams& P, float4* tab)
{
    if (threadIdx.x < 16) tab[threadIdx.x] = threadIdx.x < 8 ? P.rs_lo[threadIdx.x] : P.rs_span[threadIdx.x - 8];
}

__device__ __forceinline__ float4 reset_values_tab(const float4* tab, int b, uint4 x)
{
    const float4 lo = tab[b], sp = tab[8 + b];
    return make_float4(fmaf(sp.x, unif(x.x), lo.x), fmaf(sp.y, unif(x.y), lo.y), fmaf(sp.z, unif(x.z), lo.z),
                       fmaf(sp.w, unif(x.w), lo.w));
}

// Assemble the new episode from the sampled values of its 8 slots: state (uniform axis-angle
// quaternion, Q17), disturbance, DR factors, episode counters; the history fill value per
// rotor (Q10) in hfill.
template <uint32_t kF = kAnyFlags>
__device__ __forceinline__ void reset_finish(const DevParams& P, const float4 (&v)[8], EnvReg& e, float hfill[4])
{
    const uint32_t flags = flags_of<kF>(P);
    e.s[0] = v[0].x;
    e.s[1] = v[0].y;
    e.s[2] = v[0].z;
    const float cz = v[0].w, phi = v[1].x, th = v[1].y;
    float sxy;  // sqrt(1 - cz^2): MUFU.SQRT (relative error ~2^-23; no IEEE slow path)
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sxy) : "f"(fmaxf(fmaf(-cz, cz, 1.0f), 0.0f)));
    float sp, cp, sh, ch;
    __sincosf(phi, &sp, &cp);
    __sincosf(0.5f * th, &sh, &ch);
    e.s[3] = ch;
    e.s[4] = sh * (sxy * cp);
    e.s[5] = sh * (sxy * sp);
    e.s[6] = sh * cz;
    e.s[7] = v[1].z;
    e.s[8] = v[1].w;
    e.s[9] = v[2].x;
    e.s[10] = v[2].y;
    e.s[11] = v[2].z;
    e.s[12] = v[2].w;
    e.s[13] = v[3].x;
    e.s[14] = v[3].y;
    e.s[15] = v[3].z;
    e.s[16] = v[3].w;
    if (flags & F_DISTURBANCE) {
        e.dist[0] = v[4].x;
        e.dist[1] = v[4].y;
        e.dist[2] = v[4].z;
        e.dist[3] = v[4].w;
        e.dist[4] = v[5].x;
        e.dist[5] = v[5].y;
    } else {
#pragma unroll
        for (int j = 0; j < 6; ++j) e.dist[j] = 0.0f;
    }
    if (flags & F_DOMAIN_RAND) {
        e.dr[0] = v[6].x;
        e.dr[1] = v[6].y;
        e.dr[2] = v[6].z;
        e.dr[3] = v[6].w;
        e.dr[4] = v[7].x;
    } else {
#pragma unroll
        for (int j = 0; j < 5; ++j) e.dr[j] = 1.0f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) hfill[i] = fmaf(e.s[13 + i] - P.rpm_min, P.inv_rpm_span2, -1.0f);
    e.ep_step = 0;
    e.ep_return = 0.0f;
}

// Reset of one env from Philox counter `ctr` (thread-local draws).
__device__ __forceinline__ void reset_env(const DevParams& P, EnvReg& e, uint32_t gid, uint32_t ctr, float hfill[4])
{
    float4 v[8];
    const int nb = reset_nblocks(P);
#pragma unroll
    for (int b = 0; b < 8; ++b) v[b] = b < nb ? reset_values(P, b, reset_block(P, gid, ctr, b)) : make_float4(0, 0, 0, 0);
    reset_finish(P, v, e, hfill);  // unused DIST/DR slots are ignored
}

// Warp-cooperative reset (all 32 lanes must call; gids of a warp are consecutive): lane j of a
// round draws Philox block (j mod kNB) of reset (j / kNB) of the round and maps it to that slot's
// four sampled values; the values reach their owner through the warp's shared-memory scratch
// (kResetScratch uint4: 32 value slots + a 32-int rank->lane table).  A warp with k ending
// episodes pays ceil(k / (32 / kNB)) Philox + sampling rounds instead of kNB serial ones, and the
// owners only assemble the quaternion.  kNB = the Philox blocks of one reset that are drawn: 8
// with domain randomisation (RESET 0-3, DIST 0-1, DR 0-1), 6 without (5 resets per round; the
// DR slots stay unset and reset_finish ignores them).  Bitwise identical to reset_env (same
// integer Philox, same per-value fma).
template <int kNB, uint32_t kF = kAnyFlags>
__device__ __forceinline__ bool reset_env_warp(const DevParams& P, const float4* tab, EnvReg& e, uint32_t gid,
                                               uint32_t ctr, bool need, float hfill[4], uint4* scratch)
{
    const uint32_t flags = flags_of<kF>(P);
    static_assert(kNB == 6 || kNB == 8, "6 or 8 Philox blocks per reset");
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m == 0u) return false;
    const int lane = threadIdx.x & 31;
    constexpr int kPer = 32 / kNB;  // resets served per round
    const int nr = __popc(m);
    const int rank = __popc(m & ((1u << lane) - 1u));
    // rank -> lane table in the scratch's tail words (entries 32..39 hold 32 ints)
    int* rl = reinterpret_cast<int*>(scratch + 32);
    if (need) rl[rank] = lane;
    __syncwarp();
    const int my_q = lane / kNB, b = lane - my_q * kNB;  // reset (within the round) and slot of this lane
    const bool slot_used = b < 4 || (b < 6 && (flags & F_DISTURBANCE)) || (b >= 6 && (flags & F_DOMAIN_RAND));
    float4 v[8];
    if constexpr (kNB == 6) v[6] = v[7] = make_float4(1.f, 1.f, 1.f, 1.f);
    for (int round = 0; round * kPer < nr; ++round) {
        const int q = round * kPer + my_q;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        L2F_CHECK(nr <= 32 && rank < 32, "reset rank");
        if (my_q < kPer && q < nr && slot_used) {
            L2F_CHECK(q >= 0 && q < 32 && rl[q] >= 0 && rl[q] < 32, "reset rank->lane table");
            const uint4 blk = reset_block(P, gid - (uint32_t)lane + (uint32_t)rl[q], ctr, b);
            x = tab ? reset_values_tab(tab, b, blk) : reset_values(P, b, blk);
        }
        __syncwarp();
        reinterpret_cast<float4*>(scratch)[lane] = x;
        __syncwarp();
        if (need && rank / kPer == round) {
            const float4* src = reinterpret_cast<const float4*>(scratch) + (rank - round * kPer) * kNB;
#pragma unroll
            for (int j = 0; j < kNB; ++j) v[j] = src[j];
        }
    }
    __syncwarp();
    if (need) reset_finish<kF>(P, v, e, hfill);
    return need;
}

// Observation-noise normal i in [0,18) is normal (i mod 4) of Philox block floor(i/4) of
// stream OBS at counter t (Q20).  Blocks [b0, b1) only, so callers can spread the work.
__device__ __forceinline__ void obs_noise_blocks(const DevParams& P, uint32_t gid, uint32_t t, int b0, int b1,
                                                 float z[20])
{
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        if (b < b0 || b >= b1) continue;
        const uint4 x = draw(P, gid, t, S_OBS, (uint32_t)b);
        if (b < 4)
            box_muller2(x, z + 4 * b);
        else
            box_muller(x.x, x.y, z[4 * b], z[4 * b + 1]);
    }
}

// o += sigma (block of each component) * z: the observation noise (Q8).
__device__ __forceinline__ void add_obs_noise(const DevParams& P, const float z[20], float o[kObsCore])
{
#pragma unroll
    for (int i = 0; i < kObsCore; ++i) {
        const int g = i < 3 ? 0 : (i < 12 ? 1 : (i < 15 ? 2 : 3));
        o[i] = fmaf(P.obs_sigma[g], z[i], o[i]);
    }
}

// Noisy core observation {p, R(q) row-major, v, w} (Q8) from given normals.
template <uint32_t kF = kAnyFlags>
__device__ __forceinline__ void observe_core_z(const DevParams& P, const float* s, const float z[20],
                                               float o[kObsCore])
{
    const float qw = s[3], qx = s[4], qy = s[5], qz = s[6];
    o[0] = s[0];
    o[1] = s[1];
    o[2] = s[2];
    // R(q) with every multiply-add written out as fmaf: the compiler's own contraction of
    // a*b +- c*d may pick either product, and differently in two builds of this function
    // (seen between the debug-check build's specialised and generic step kernels)
    const float x2 = qx + qx, y2 = qy + qy, z2 = qz + qz;  // exact doublings
    const float wx2 = qw * x2, wy2 = qw * y2, wz2 = qw * z2;
    o[3] = fmaf(-qy, y2, fmaf(-qz, z2, 1.0f));
    o[4] = fmaf(qx, y2, -wz2);
    o[5] = fmaf(qx, z2, wy2);
    o[6] = fmaf(qx, y2, wz2);
    o[7] = fmaf(-qx, x2, fmaf(-qz, z2, 1.0f));
    o[8] = fmaf(qy, z2, -wx2);
    o[9] = fmaf(qx, z2, -wy2);
    o[10] = fmaf(qy, z2, wx2);
    o[11] = fmaf(-qx, x2, fmaf(-qy, y2, 1.0f));
    o[12] = s[7];
    o[13] = s[8];
    o[14] = s[9];
    o[15] = s[10];
    o[16] = s[11];
    o[17] = s[12];
    if (flags_of<kF>(P) & F_OBS_NOISE) add_obs_noise(P, z, o);
}

template <uint32_t kF = kAnyFlags>
__device__ __forceinline__ void observe_core(const DevParams& P, const float* s, uint32_t gid, uint32_t t,
                                             float o[kObsCore])
{
    float z[20];
    if (flags_of<kF>(P) & F_OBS_NOISE) obs_noise_blocks(P, gid, t, 0, 5, z);
    observe_core_z<kF>(P, s, z, o);
}

// Logical history entry H[k] (k-th most recent action, most recent first) at step t:
// tau = t - 1 - k; ring slot (tau mod N_H) if tau >= hist_t0, else the episode's fill value.
__device__ __forceinline__ void hist_entry(const DevBufs& B, int64_t N, int n_hist, int64_t i, int64_t t, int k,
                                           int32_t t0, float h[4])
{
    const int64_t tau = t - 1 - k;
    L2F_CHECK(i >= 0 && i < N && k >= 0 && k < n_hist, "hist_entry index");
    if (tau >= (int64_t)t0) {
        const int slot = (int)(((tau % n_hist) + n_hist) % n_hist);
        const float4 v = B.hist[(int64_t)slot * N + i];
        h[0] = v.x, h[1] = v.y, h[2] = v.z, h[3] = v.w;
    } else {
        const float4 v = B.hist_fill[i];
        h[0] = v.x, h[1] = v.y, h[2] = v.z, h[3] = v.w;
    }
}

// Open-loop random action (stream RAND_ACT): a_i = -1 + 2 u_i.
__device__ __forceinline__ void random_action(const DevParams& P, uint32_t gid, uint32_t t, float a[4])
{
    const uint4 x = draw(P, gid, t, S_RAND_ACT, 0);
    a[0] = uab(-1.0f, 1.0f, x.x);
    a[1] = uab(-1.0f, 1.0f, x.y);
    a[2] = uab(-1.0f, 1.0f, x.z);
    a[3] = uab(-1.0f, 1.0f, x.w);
}

// ---------------------------------------------------------------------------------------
// Episode statistics: per-thread accumulation -> warp (REDUX / shuffles) -> block partial
// in a fixed order -> the block's slot (deterministic for a fixed launch sequence).
// ---------------------------------------------------------------------------------------
struct StatAcc {
    int32_t ep, term, trunc, div, len;
    double ret, ret2;
};

__device__ __forceinline__ void stat_zero(StatAcc& a)
{
    a.ep = a.term = a.trunc = a.div = a.len = 0;
    a.ret = a.ret2 = 0.0;
}

__device__ __forceinline__ void stat_episode(StatAcc& a, const Trans& o)
{
    a.ep += 1;
    a.term += (o.flags & D_TERM) ? 1 : 0;
    a.trunc += (o.flags & D_TRUNC) ? 1 : 0;
    a.div += (o.flags & D_DIV) ? 1 : 0;
    a.len += o.len;
    const double r = (double)o.ret;
    a.ret += r;
    a.ret2 += r * r;
}

// Compact per-thread accumulator of one rollout unit (at most 65535 steps per thread between
// flushes): (episodes | terminated << 16), (truncated | diverged << 16), summed lengths, and the
// unit's return sums in FP32 (a unit of T <= 65535 steps ends at most T episodes per env; the
// per-unit sums go to FP64 at the flush, so FP32 only carries one env's ~T / 9 returns: relative
// error ~1e-6 in the reported return moments) -- 5 registers, no FP64 in the step loop.
struct StatPk {
    uint32_t ep_term, trunc_div, len;
    float ret, ret2;
};

__device__ __forceinline__ void statpk_zero(StatPk& a)
{
    a.ep_term = a.trunc_div = a.len = 0u;
    a.ret = a.ret2 = 0.0f;
}

// Branch-free update: `ended` selects whether the transition closed an episode.
__device__ __forceinline__ void statpk_episode(StatPk& a, const Trans& o, bool ended)
{
    a.ep_term += ended ? 1u + ((o.flags & D_TERM) ? 0x10000u : 0u) : 0u;
    a.trunc_div += ended ? ((o.flags & D_TRUNC) ? 1u : 0u) + ((o.flags & D_DIV) ? 0x10000u : 0u) : 0u;
    a.len += ended ? (uint32_t)o.len : 0u;
    const float r = ended ? o.ret : 0.0f;
    a.ret += r;
    a.ret2 = fmaf(r, r, a.ret2);
}

__device__ __forceinline__ StatAcc statpk_unpack(const StatPk& a)
{
    StatAcc r;
    r.ep = (int32_t)(a.ep_term & 0xFFFFu);
    r.term = (int32_t)(a.ep_term >> 16);
    r.trunc = (int32_t)(a.trunc_div & 0xFFFFu);
    r.div = (int32_t)(a.trunc_div >> 16);
    r.len = (int32_t)a.len;
    r.ret = (double)a.ret;
    r.ret2 = (double)a.ret2;
    return r;
}

// Warp-reduce a unit's accumulator (fixed shuffle order) and add it, with `steps` env-steps, to
// the warp's FP64 row (lane 0 writes).  All 32 lanes must call it.
__device__ __forceinline__ void statpk_flush(const StatPk& a, double steps, double* row)
{
    const unsigned m = 0xffffffffu;
    const uint32_t ep = __reduce_add_sync(m, a.ep_term & 0xFFFFu), term = __reduce_add_sync(m, a.ep_term >> 16);
    const uint32_t tr = __reduce_add_sync(m, a.trunc_div & 0xFFFFu), dv = __reduce_add_sync(m, a.trunc_div >> 16);
    const uint32_t len = __reduce_add_sync(m, a.len);
    double r = (double)a.ret, r2 = (double)a.ret2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(m, r, o);
        r2 += __shfl_xor_sync(m, r2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        row[0] += ep;
        row[1] += term;
        row[2] += tr;
        row[3] += dv;
        row[4] += len;
        row[5] += r;
        row[6] += r2;
        row[7] += steps;
    }
}

// Warp-reduce a StatPk (integer REDUX, FP32 shuffles in a fixed order) and write lane 0's
// result as FP64 into smem row[8]; row[7] = 0.  All 32 lanes must call it.
__device__ __forceinline__ void statpk_warp_to_smem(const StatPk& a, double* row)
{
    const unsigned m = 0xffffffffu;
    const uint32_t ep = __reduce_add_sync(m, a.ep_term & 0xFFFFu), term = __reduce_add_sync(m, a.ep_term >> 16);
    const uint32_t tr = __reduce_add_sync(m, a.trunc_div & 0xFFFFu), dv = __reduce_add_sync(m, a.trunc_div >> 16);
    const uint32_t len = __reduce_add_sync(m, a.len);
    float r = a.ret, r2 = a.ret2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(m, r, o);
        r2 += __shfl_xor_sync(m, r2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        row[0] = ep;
        row[1] = term;
        row[2] = tr;
        row[3] = dv;
        row[4] = len;
        row[5] = r;
        row[6] = r2;
        row[7] = 0.0;
    }
}

// Warp-reduce `a` and write lane 0's result into smem[warp][8] (doubles); returns nothing.
// All 32 lanes must call it.
__device__ __forceinline__ void stat_warp_to_smem(const StatAcc& a, double* smem_warp_row)
{
    const unsigned m = 0xffffffffu;
    const int ep = __reduce_add_sync(m, a.ep);
    const int term = __reduce_add_sync(m, a.term);
    const int trunc = __reduce_add_sync(m, a.trunc);
    const int dv = __reduce_add_sync(m, a.div);
    const int len = __reduce_add_sync(m, a.len);
    double r = a.ret, r2 = a.ret2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(m, r, o);
        r2 += __shfl_xor_sync(m, r2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        smem_warp_row[0] = ep;
        smem_warp_row[1] = term;
        smem_warp_row[2] = trunc;
        smem_warp_row[3] = dv;
        smem_warp_row[4] = len;
        smem_warp_row[5] = r;
        smem_warp_row[6] = r2;
        smem_warp_row[7] = 0.0;
    }
}

// Fixed-order sum of nw warp rows into slot[0..6] plus `steps` into slot[7].  Call after a
// barrier that makes the warp rows visible; threads 0..7 participate.
__device__ __forceinline__ void stat_rows_to_slot(const double* smem, int nw, double steps, double* slot)
{
    if (threadIdx.x < kStatsLen) {
        double x = 0.0;
        if (threadIdx.x < 7)
            for (int w = 0; w < nw; ++w) x += smem[w * kStatsLen + threadIdx.x];
        else
            x = steps;
        slot[threadIdx.x] += x;
    }
}

}  // namespace l2f
