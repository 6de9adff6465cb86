// l2f_td3.cu -- GPU-batched TD3 update ("we use TD3", S:368-455;
// DESIGN.md Q32-Q35), sm_100a.
//
// One CTA per agent, one thread per batch sample (B <= 256): many independent agents (seeds,
// ablation configurations -- the paper's Table II runs 10 configurations x 50 seeds) are
// updated concurrently, one per SM.  FP32 master weights in a flat per-agent block:
//   [actor, actor', Q1, Q2, Q1', Q2', m_actor, v_actor, m_Q1, v_Q1, m_Q2, v_Q2]
// each net W1[hid][in], b1, W2[hid][hid], b2, W3[out][hid], b3 (the oracle's layout; the actor
// part is the l2f_policy layout, so it exports to the tcgen05 rollout after fp16 rounding).
//
// Per update: (1) target actions with clipped smoothing noise and the clipped double-Q target
// y; (2) per critic: forward with cached activations, per-sample deltas, weight gradients as
// D^T X reductions over the batch, Adam; (3) on delayed steps the deterministic policy
// gradient through the updated Q1's action input, Adam, Polyak averaging of the targets.
//
// Layout of the work: the weights of the net in use are staged in shared memory (rows padded
// to a multiple of 4 floats), the actor input rows too; each thread keeps its sample's
// hidden vectors in registers (fully unrolled 64-wide loops, float4 weight reads that every
// lane of a warp takes from the same address -- one shared-memory wavefront), and writes the
// per-sample rows the weight gradients need to a per-agent global scratch (L2-resident).
#include <cmath>

#include "l2f_internal.h"

namespace l2f {
namespace {

constexpr int kT = 256;   // threads = max batch
constexpr int kH = 64;    // hidden width
constexpr int kCI = 32;   // critic input: o_c (28) + a (4)

__host__ __device__ constexpr int net_size(int in, int out) { return kH * in + kH + kH * kH + kH + out * kH + out; }
__host__ __device__ constexpr int pad4(int k) { return (k + 3) & ~3; }

struct NetP {  // views into a flat parameter block (global)
    float *W1, *b1, *W2, *b2, *W3, *b3;
    int in, out;
};

__device__ __forceinline__ NetP net_at(float* p, int in, int out)
{
    NetP n;
    n.in = in;
    n.out = out;
    n.W1 = p;
    p += kH * in;
    n.b1 = p;
    p += kH;
    n.W2 = p;
    p += kH * kH;
    n.b2 = p;
    p += kH;
    n.W3 = p;
    p += out * kH;
    n.b3 = p;
    return n;
}

// A net staged in shared memory: W1 rows padded to ld1 = pad4(in); W2, W3 rows of 64.
struct NetS {
    float *W1, *b1, *W2, *b2, *W3, *b3;
    int in, ld1, out;
};

__host__ __device__ constexpr int stage_floats(int in, int out)
{
    return kH * pad4(in) + kH + kH * kH + kH + out * kH + 4;
}

// CTA-cooperative copy of a net into shared memory at sm (16-byte aligned); caller syncs.
__device__ NetS stage(const NetP& n, float* sm)
{
    NetS S;
    S.in = n.in;
    S.out = n.out;
    S.ld1 = pad4(n.in);
    S.W1 = sm;
    S.b1 = S.W1 + kH * S.ld1;
    S.W2 = S.b1 + kH;
    S.b2 = S.W2 + kH * kH;
    S.W3 = S.b2 + kH;
    S.b3 = S.W3 + n.out * kH;
#pragma unroll 4
    for (int e = threadIdx.x; e < kH * S.ld1; e += blockDim.x) {
        const int j = e / S.ld1, i = e - j * S.ld1;
        S.W1[e] = i < n.in ? n.W1[j * n.in + i] : 0.0f;
    }
#pragma unroll 4
    for (int e = threadIdx.x; e < kH * kH; e += blockDim.x) S.W2[e] = n.W2[e];
    for (int e = threadIdx.x; e < n.out * kH; e += blockDim.x) S.W3[e] = n.W3[e];
    for (int e = threadIdx.x; e < kH; e += blockDim.x) {
        S.b1[e] = n.b1[e];
        S.b2[e] = n.b2[e];
    }
    if ((int)threadIdx.x < n.out) S.b3[threadIdx.x] = n.b3[threadIdx.x];
    return S;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Compiler scheduling fence: keeps the fully unrolled 64-wide loops from hoisting hundreds of
// shared-memory loads ahead (which spills), without emitting an instruction.
__device__ __forceinline__ void sched_fence() { asm volatile("" ::: "memory"); }

__device__ __forceinline__ void fma4(float& acc, float4 w, float4 x)
{
    acc = fmaf(w.x, x.x, acc);
    acc = fmaf(w.y, x.y, acc);
    acc = fmaf(w.z, x.z, acc);
    acc = fmaf(w.w, x.w, acc);
}

// h = relu(W1 x + b1) with x a shared-memory row of S.ld1 floats (padded with zeros); 16
// outputs per pass over the row (x re-read 4 times, 16 accumulators live).
__device__ __forceinline__ void layer1_smem(const NetS& S, const float* x, float (&h)[kH])
{
#pragma unroll
    for (int jb = 0; jb < kH; jb += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = S.b1[jb + j];
#pragma unroll 1
        for (int c = 0; c < S.ld1; c += 4) {
            const float4 xv = ld4(x + c);
#pragma unroll
            for (int j = 0; j < 16; ++j) fma4(acc[j], ld4(S.W1 + (jb + j) * S.ld1 + c), xv);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) h[jb + j] = fmaxf(acc[j], 0.0f);
    }
}

// h = relu(W1 x + b1) with x the 32-float critic input in registers (ld1 = 32).
__device__ __forceinline__ void layer1_reg(const NetS& S, const float (&x)[kCI], float (&h)[kH])
{
#pragma unroll
    for (int j = 0; j < kH; ++j) {
        float acc = S.b1[j];
#pragma unroll
        for (int c = 0; c < kCI; c += 4)
            fma4(acc, ld4(S.W1 + j * kCI + c), make_float4(x[c], x[c + 1], x[c + 2], x[c + 3]));
        h[j] = fmaxf(acc, 0.0f);
        if (j % 8 == 7) sched_fence();
    }
}

// h2 = relu(W2 h1 + b2)
__device__ __forceinline__ void layer2(const NetS& S, const float (&h1)[kH], float (&h2)[kH])
{
#pragma unroll
    for (int j = 0; j < kH; ++j) {
        float acc = S.b2[j];
#pragma unroll
        for (int c = 0; c < kH; c += 4)
            fma4(acc, ld4(S.W2 + j * kH + c), make_float4(h1[c], h1[c + 1], h1[c + 2], h1[c + 3]));
        h2[j] = fmaxf(acc, 0.0f);
        if (j % 4 == 3) sched_fence();
    }
}

// y = W3 h2 + b3 (OUT outputs), tanh optional
template <int OUT>
__device__ __forceinline__ void layer3(const NetS& S, const float (&h2)[kH], float (&y)[OUT], bool tanh_out)
{
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
        float acc = S.b3[o];
#pragma unroll
        for (int c = 0; c < kH; c += 4)
            fma4(acc, ld4(S.W3 + o * kH + c), make_float4(h2[c], h2[c + 1], h2[c + 2], h2[c + 3]));
        y[o] = tanh_out ? tanhf(acc) : acc;
    }
}

// d2 = (W3^T d3) o relu'(h2)
template <int OUT>
__device__ __forceinline__ void delta2(const NetS& S, const float (&d3)[OUT], const float (&h2)[kH], float (&d2)[kH])
{
#pragma unroll
    for (int j = 0; j < kH; ++j) {
        float acc = 0.0f;
#pragma unroll
        for (int o = 0; o < OUT; ++o) acc = fmaf(S.W3[o * kH + j], d3[o], acc);
        d2[j] = h2[j] > 0.0f ? acc : 0.0f;
    }
}

// d1 = (W2^T d2) o relu'(h1), four outputs at a time (float4 column slices of the W2 rows),
// so only d2 and four accumulators are live.  d1 may alias h1.
__device__ __forceinline__ void delta1(const NetS& S, const float (&d2)[kH], float (&h1_d1)[kH])
{
#pragma unroll
    for (int c = 0; c < kH; c += 4) {
        float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
        for (int j = 0; j < kH; ++j) {
            const float4 w = ld4(S.W2 + j * kH + c);
            a0 = fmaf(w.x, d2[j], a0);
            a1 = fmaf(w.y, d2[j], a1);
            a2 = fmaf(w.z, d2[j], a2);
            a3 = fmaf(w.w, d2[j], a3);
        }
        h1_d1[c] = h1_d1[c] > 0.0f ? a0 : 0.0f;
        h1_d1[c + 1] = h1_d1[c + 1] > 0.0f ? a1 : 0.0f;
        h1_d1[c + 2] = h1_d1[c + 2] > 0.0f ? a2 : 0.0f;
        h1_d1[c + 3] = h1_d1[c + 3] > 0.0f ? a3 : 0.0f;
        sched_fence();
    }
}

__device__ __forceinline__ void store_row(float* dst, const float (&v)[kH])
{
#pragma unroll
    for (int c = 0; c < kH; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
}
__device__ __forceinline__ void load_row(const float* src, float (&v)[kH])
{
#pragma unroll
    for (int c = 0; c < kH; c += 4) {
        const float4 x = ld4(src + c);
        v[c] = x.x;
        v[c + 1] = x.y;
        v[c + 2] = x.z;
        v[c + 3] = x.w;
    }
}

// Weight gradient of one layer, reduced over the batch: gW[j][i] = sum_s D[s][j] X[s][i] (gW
// row stride K, unpadded: the parameter layout), gb[j] = sum_s D[s][j].  CTA-cooperative,
// 4 x 4 register tiles; D rows (ldd) and X rows (ldx) 16-byte aligned, ldx >= pad4(K) with
// zero padding.
__device__ void grad_layer(const float* D, int ldd, const float* X, int ldx, int B, int N, int K, float* gW,
                           float* gb)
{
    const int tj = (N + 3) / 4, ti = (K + 3) / 4;
    for (int tile = threadIdx.x; tile < tj * ti; tile += blockDim.x) {
        const int j0 = (tile / ti) * 4, i0 = (tile % ti) * 4;
        float acc[4][4] = {};
        if (N % 4 == 0) {
#pragma unroll 8
            for (int s = 0; s < B; ++s) {
                const float4 d = ld4(D + s * ldd + j0), x = ld4(X + s * ldx + i0);
                const float dv[4] = {d.x, d.y, d.z, d.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(dv[a], xv[b], acc[a][b]);
            }
        } else {  // N = 1 (the critic's output layer)
#pragma unroll 8
            for (int s = 0; s < B; ++s) {
                const float d = D[s * ldd + j0];
                const float4 x = ld4(X + s * ldx + i0);
                acc[0][0] = fmaf(d, x.x, acc[0][0]);
                acc[0][1] = fmaf(d, x.y, acc[0][1]);
                acc[0][2] = fmaf(d, x.z, acc[0][2]);
                acc[0][3] = fmaf(d, x.w, acc[0][3]);
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (j0 + a < N && i0 + b < K) gW[(j0 + a) * K + i0 + b] = acc[a][b];
    }
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        float acc = 0.0f;
#pragma unroll 8
        for (int s = 0; s < B; ++s) acc += D[s * ldd + j];
        gb[j] = acc;
    }
}

struct AdamC {
    float lr, b1, b2, c1, c2, eps;  // c1 = 1 - beta1^t, c2 = 1 - beta2^t
};

__device__ void adam(float* th, float* m, float* v, const float* g, int n, const AdamC& A)
{
#pragma unroll 4
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const float gk = g[k];
        const float mk = fmaf(A.b1, m[k], (1.0f - A.b1) * gk);
        const float vk = fmaf(A.b2, v[k], (1.0f - A.b2) * gk * gk);
        m[k] = mk;
        v[k] = vk;
        th[k] -= A.lr * (mk / A.c1) / (sqrtf(vk / A.c2) + A.eps);
    }
}

__device__ __forceinline__ float block_sum(float x, float* red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    float t = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

// Scratch layout per agent (floats): per-sample rows (16-byte aligned) then the raw gradients
// [Q1, Q2, actor] of the last update (read by the tests through TD3.grads(): they start at
// B x 554 floats).
struct TD3Scratch {
    float *xc, *h1, *h2, *d1, *d2, *ah1, *ah2, *ad1, *ad2, *aout, *ad3, *y, *d3, *gq1, *gq2, *ga;
};

__host__ __device__ inline int64_t td3_scratch_floats(int in_dim, int B)
{
    const int64_t f = (int64_t)B * (kCI + 8 * kH + 4 + 4 + 1 + 1) + 2 * net_size(kCI, 1) + net_size(in_dim, 4);
    return (f + 63) & ~(int64_t)63;  // every agent's scratch 256-byte aligned (float4 rows)
}

__device__ inline TD3Scratch scratch_at(float* p, int B)
{
    TD3Scratch S;
    S.xc = p;  // [B][32]
    p += B * kCI;
    S.h1 = p;  // [B][64] ...
    p += B * kH;
    S.h2 = p;
    p += B * kH;
    S.d1 = p;
    p += B * kH;
    S.d2 = p;
    p += B * kH;
    S.ah1 = p;
    p += B * kH;
    S.ah2 = p;
    p += B * kH;
    S.ad1 = p;
    p += B * kH;
    S.ad2 = p;
    p += B * kH;
    S.aout = p;  // [B][4]
    p += B * 4;
    S.ad3 = p;  // [B][4]
    p += B * 4;
    S.y = p;  // [B]
    p += B;
    S.d3 = p;  // [B]
    p += B;
    S.gq1 = p;
    p += net_size(kCI, 1);
    S.gq2 = p;
    p += net_size(kCI, 1);
    S.ga = p;
    return S;
}

__global__ void __launch_bounds__(kT, 1) td3_update_kernel(TD3Dev A)
{
    extern __shared__ __align__(16) float sm[];
    __shared__ float red[kT / 32];
    const int ag = blockIdx.x, B = A.B, I = A.in_dim, s = threadIdx.x, LI = pad4(A.in_dim);
    const bool act = s < B;
    const int na = net_size(I, 4), nc = net_size(kCI, 1);
    float* P = A.params + (int64_t)ag * A.block;
    NetP actor = net_at(P, I, 4), actor_t = net_at(P + na, I, 4);
    NetP Q[2] = {net_at(P + 2 * na, kCI, 1), net_at(P + 2 * na + nc, kCI, 1)};
    NetP Qt[2] = {net_at(P + 2 * na + 2 * nc, kCI, 1), net_at(P + 2 * na + 3 * nc, kCI, 1)};
    float* m_a = P + 2 * na + 4 * nc;
    float* v_a = m_a + na;
    float* m_c[2] = {v_a + na, v_a + na + 2 * nc};
    float* v_c[2] = {v_a + na + nc, v_a + na + 3 * nc};
    TD3Scratch S = scratch_at(A.scratch + (int64_t)ag * A.scratch_floats, B);
    const int64_t rb = (int64_t)ag * B + s;  // this sample's row in the [A][B][...] batch arrays
    // shared memory: input rows xs [B][LI], then one staged net
    float* xs = sm;
    float* wsm = sm + pad4(B * LI);
    float h1[kH], h2[kH], x[kCI];

    // ---- 1. target: a' = clip(pi'(o_a') + clip(sigma eps, -c, c), -1, 1); y = r + g (1-d) min Q'
#pragma unroll 4
    for (int e = threadIdx.x; e < B * LI; e += blockDim.x) {
        const int r = e / LI, i = e - r * LI;
        xs[e] = i < I ? A.o_a2[((int64_t)ag * B + r) * I + i] : 0.0f;
    }
    NetS W = stage(actor_t, wsm);
    __syncthreads();
    if (act) {
        float at[4];
        layer1_smem(W, xs + s * LI, h1);
        layer2(W, h1, h2);
        layer3<4>(W, h2, at, true);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float nz = fminf(fmaxf(A.sigma_t * A.eps[rb * 4 + k], -A.clip_t), A.clip_t);
            at[k] = fminf(fmaxf(at[k] + nz, -1.0f), 1.0f);
        }
#pragma unroll
        for (int k = 0; k < 28; ++k) x[k] = A.o_c2[rb * 28 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[28 + k] = at[k];
    }
    float qmin = 0.0f;
    for (int c = 0; c < 2; ++c) {
        __syncthreads();
        W = stage(Qt[c], wsm);
        __syncthreads();
        if (act) {
            float q[1];
            layer1_reg(W, x, h1);
            layer2(W, h1, h2);
            layer3<1>(W, h2, q, false);
            qmin = c == 0 ? q[0] : fminf(qmin, q[0]);
        }
    }
    float y = 0.0f;
    if (act) {
        y = A.r[rb] + A.gamma * (1.0f - A.done[rb]) * qmin;
        // the critic input (o_c, a) of this sample, shared by both critics
#pragma unroll
        for (int k = 0; k < 28; ++k) x[k] = A.o_c[rb * 28 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[28 + k] = A.a[rb * 4 + k];
#pragma unroll
        for (int k = 0; k < kCI; k += 4)
            *reinterpret_cast<float4*>(S.xc + s * kCI + k) = make_float4(x[k], x[k + 1], x[k + 2], x[k + 3]);
    }

    // ---- 2. critics: MSE to y, Adam
    const AdamC Ac{A.lr_critic, A.beta1, A.beta2, A.c1_critic, A.c2_critic, A.adam_eps};
    for (int c = 0; c < 2; ++c) {
        __syncthreads();
        W = stage(Q[c], wsm);
        __syncthreads();
        float lossc = 0.0f;
        if (act) {
            float q[1], d2[kH];
            layer1_reg(W, x, h1);
            store_row(S.h1 + s * kH, h1);
            layer2(W, h1, h2);
            store_row(S.h2 + s * kH, h2);
            layer3<1>(W, h2, q, false);
            const float e = q[0] - y;
            lossc = e * e / (float)B;
            const float d3[1] = {2.0f * e / (float)B};
            delta2<1>(W, d3, h2, d2);
            store_row(S.d2 + s * kH, d2);
            delta1(W, d2, h1);  // h1 <- d1
            store_row(S.d1 + s * kH, h1);
            S.d3[s] = d3[0];
        }
        const float loss = block_sum(lossc, red);
        if (threadIdx.x == 0) A.losses[ag * 3 + c] = loss;
        __syncthreads();
        float* g = c == 0 ? S.gq1 : S.gq2;
        NetP gn = net_at(g, kCI, 1);
        grad_layer(S.d1, kH, S.xc, kCI, B, kH, kCI, gn.W1, gn.b1);
        grad_layer(S.d2, kH, S.h1, kH, B, kH, kH, gn.W2, gn.b2);
        grad_layer(S.d3, 1, S.h2, kH, B, 1, kH, gn.W3, gn.b3);
        __syncthreads();
        adam(Q[c].W1, m_c[c], v_c[c], g, nc, Ac);
    }
    if (!A.update_actor) {
        if (threadIdx.x == 0) A.losses[ag * 3 + 2] = 0.0f;
        return;
    }

    // ---- 3. actor: ascend Q1(o_c, pi(o_a)) through the updated Q1's action input, Adam
    __syncthreads();
#pragma unroll 4
    for (int e = threadIdx.x; e < B * LI; e += blockDim.x) {
        const int r = e / LI, i = e - r * LI;
        xs[e] = i < I ? A.o_a[((int64_t)ag * B + r) * I + i] : 0.0f;
    }
    W = stage(actor, wsm);
    __syncthreads();
    float ap[4] = {0.f, 0.f, 0.f, 0.f};
    if (act) {
        layer1_smem(W, xs + s * LI, h1);
        store_row(S.ah1 + s * kH, h1);
        layer2(W, h1, h2);
        store_row(S.ah2 + s * kH, h2);
        layer3<4>(W, h2, ap, true);
#pragma unroll
        for (int k = 0; k < 4; ++k) x[28 + k] = ap[k];
    }
    __syncthreads();
    W = stage(Q[0], wsm);  // the updated Q1
    __syncthreads();
    float lossa = 0.0f;
    float da[4] = {0.f, 0.f, 0.f, 0.f};
    if (act) {
        float q[1], d2[kH];
        layer1_reg(W, x, h1);
        layer2(W, h1, h2);
        layer3<1>(W, h2, q, false);
        lossa = -q[0] / (float)B;
        const float d3[1] = {-1.0f / (float)B};
        delta2<1>(W, d3, h2, d2);
        delta1(W, d2, h1);  // h1 <- d1 of Q1
        // dL/da = (W1^T d1)[28..31]
#pragma unroll
        for (int j = 0; j < kH; ++j) {
            const float4 w = ld4(W.W1 + j * kCI + 28);
            da[0] = fmaf(w.x, h1[j], da[0]);
            da[1] = fmaf(w.y, h1[j], da[1]);
            da[2] = fmaf(w.z, h1[j], da[2]);
            da[3] = fmaf(w.w, h1[j], da[3]);
        }
    }
    __syncthreads();
    W = stage(actor, wsm);
    __syncthreads();
    if (act) {
        float d3a[4], e2[kH];
#pragma unroll
        for (int k = 0; k < 4; ++k) d3a[k] = da[k] * (1.0f - ap[k] * ap[k]);
        load_row(S.ah2 + s * kH, h2);
        delta2<4>(W, d3a, h2, e2);
        store_row(S.ad2 + s * kH, e2);
        load_row(S.ah1 + s * kH, h1);
        delta1(W, e2, h1);  // h1 <- actor d1
        store_row(S.ad1 + s * kH, h1);
        *reinterpret_cast<float4*>(S.ad3 + s * 4) = make_float4(d3a[0], d3a[1], d3a[2], d3a[3]);
    }
    const float loss = block_sum(lossa, red);
    if (threadIdx.x == 0) A.losses[ag * 3 + 2] = loss;
    __syncthreads();
    NetP ga = net_at(S.ga, I, 4);
    grad_layer(S.ad1, kH, xs, LI, B, kH, I, ga.W1, ga.b1);
    grad_layer(S.ad2, kH, S.ah1, kH, B, kH, kH, ga.W2, ga.b2);
    grad_layer(S.ad3, 4, S.ah2, kH, B, 4, kH, ga.W3, ga.b3);
    __syncthreads();
    const AdamC Aa{A.lr_actor, A.beta1, A.beta2, A.c1_actor, A.c2_actor, A.adam_eps};
    adam(actor.W1, m_a, v_a, S.ga, na, Aa);
    __syncthreads();
    // ---- 4. Polyak averaging of the three targets
    const float tau = A.tau;
#pragma unroll 4
    for (int k = threadIdx.x; k < na; k += blockDim.x)
        actor_t.W1[k] = fmaf(tau, actor.W1[k], (1.0f - tau) * actor_t.W1[k]);
    for (int c = 0; c < 2; ++c)
#pragma unroll 4
        for (int k = threadIdx.x; k < nc; k += blockDim.x) Qt[c].W1[k] = fmaf(tau, Q[c].W1[k], (1.0f - tau) * Qt[c].W1[k]);
}

size_t td3_smem_bytes(int in_dim, int B)
{
    const int a = stage_floats(in_dim, 4), c = stage_floats(kCI, 1);
    return (size_t)(pad4(B * pad4(in_dim)) + (a > c ? a : c)) * sizeof(float);
}

}  // namespace

int64_t td3_block_floats(int in_dim) { return 4 * (int64_t)net_size(in_dim, 4) + 8 * (int64_t)net_size(kCI, 1); }
int64_t td3_scratch_bytes(int in_dim, int B) { return 4 * td3_scratch_floats(in_dim, B); }

cudaError_t launch_td3_update(const TD3Dev& A, cudaStream_t s)
{
    if (A.B < 1 || A.B > kT || A.in_dim < 1 || A.in_dim > 256) return cudaErrorNotSupported;
    const size_t smem = td3_smem_bytes(A.in_dim, A.B);
    if (smem > 220 * 1024) return cudaErrorNotSupported;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(td3_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    td3_update_kernel<<<A.n_agents, kT, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace l2f
