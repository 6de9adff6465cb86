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
// y; (2) per critic: forward with cached activations, per-sample deltas (thread-local),
// weight gradients as D^T X reductions over the batch (register-tiled, CTA-wide), Adam; (3) on
// delayed steps the deterministic policy gradient through the updated Q1's action input, Adam,
// Polyak averaging of the three targets.  Per-sample rows live in a per-agent global scratch
// (L2-resident); the current input rows in shared memory.
#include <cmath>

#include "l2f_internal.h"

namespace l2f {
namespace {

constexpr int kT = 256;   // threads = max batch
constexpr int kH = 64;    // hidden width
constexpr int kCI = 32;   // critic input: o_c (28) + a (4)

struct NetP {  // views into a flat parameter block
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

__host__ __device__ constexpr int net_size(int in, int out) { return kH * in + kH + kH * kH + kH + out * kH + out; }

// Forward of one sample: x (in) -> h1, h2 (post-ReLU) -> y (out), tanh or linear output.
// Weights are read by all threads at the same addresses (broadcast through L1).
__device__ __forceinline__ void fwd(const NetP& n, const float* x, float* h1, float* h2, float* y, bool tanh_out)
{
    for (int j = 0; j < kH; ++j) {
        const float* w = n.W1 + j * n.in;
        float acc = n.b1[j];
        for (int i = 0; i < n.in; ++i) acc = fmaf(w[i], x[i], acc);
        h1[j] = fmaxf(acc, 0.0f);
    }
    for (int j = 0; j < kH; ++j) {
        const float* w = n.W2 + j * kH;
        float acc = n.b2[j];
#pragma unroll 8
        for (int i = 0; i < kH; ++i) acc = fmaf(w[i], h1[i], acc);
        h2[j] = fmaxf(acc, 0.0f);
    }
    for (int o = 0; o < n.out; ++o) {
        const float* w = n.W3 + o * kH;
        float acc = n.b3[o];
#pragma unroll 8
        for (int i = 0; i < kH; ++i) acc = fmaf(w[i], h2[i], acc);
        y[o] = tanh_out ? tanhf(acc) : acc;
    }
}

// Per-sample backward deltas: d3 (out, already through the output activation) -> d2, d1 (after
// ReLU'), and dx = W1^T d1 if dx != nullptr.
__device__ __forceinline__ void bwd_deltas(const NetP& n, const float* h1, const float* h2, const float* d3,
                                           float* d2, float* d1, float* dx)
{
    for (int j = 0; j < kH; ++j) {
        float acc = 0.0f;
        for (int o = 0; o < n.out; ++o) acc = fmaf(n.W3[o * kH + j], d3[o], acc);
        d2[j] = h2[j] > 0.0f ? acc : 0.0f;
    }
    for (int i = 0; i < kH; ++i) {
        float acc = 0.0f;
#pragma unroll 8
        for (int j = 0; j < kH; ++j) acc = fmaf(n.W2[j * kH + i], d2[j], acc);
        d1[i] = h1[i] > 0.0f ? acc : 0.0f;
    }
    if (dx)
        for (int i = 0; i < n.in; ++i) {
            float acc = 0.0f;
#pragma unroll 8
            for (int j = 0; j < kH; ++j) acc = fmaf(n.W1[j * n.in + i], d1[j], acc);
            dx[i] = acc;
        }
}

// Weight gradient of one layer, reduced over the batch: gW[j][i] = sum_s D[s][j] X[s][i],
// gb[j] = sum_s D[s][j].  CTA-cooperative, 4 x 4 register tiles per thread.
__device__ void grad_layer(const float* D, int ldd, const float* X, int ldx, int B, int N, int K, float* gW,
                           float* gb)
{
    const int tj = (N + 3) / 4, ti = (K + 3) / 4;
    for (int tile = threadIdx.x; tile < tj * ti; tile += blockDim.x) {
        const int j0 = (tile / ti) * 4, i0 = (tile % ti) * 4;
        float acc[4][4] = {};
        for (int s = 0; s < B; ++s) {
            float d[4], x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                d[q] = j0 + q < N ? D[s * ldd + j0 + q] : 0.0f;
                x[q] = i0 + q < K ? X[s * ldx + i0 + q] : 0.0f;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(d[a], x[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (j0 + a < N && i0 + b < K) gW[(j0 + a) * K + i0 + b] = acc[a][b];
    }
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < B; ++s) acc += D[s * ldd + j];
        gb[j] = acc;
    }
}

struct AdamC {
    float lr, b1, b2, c1, c2, eps;  // c1 = 1 - beta1^t, c2 = 1 - beta2^t
};

__device__ void adam(float* th, float* m, float* v, const float* g, int n, const AdamC& A)
{
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

}  // namespace

// Scratch layout per agent (floats), see l2f_td3_sizes.
struct TD3Scratch {
    float *y, *xc, *h1, *h2, *d1, *d2, *d3, *ah1, *ah2, *aout, *ad1, *ad2, *ad3, *gq1, *gq2, *ga;
};

__host__ __device__ inline int64_t td3_scratch_floats(int in_dim, int B)
{
    (void)in_dim;
    return (int64_t)B * (1 + kCI + 4 * kH + 1 + 2 * kH + 4 + 2 * kH + 4) + 2 * net_size(kCI, 1) +
           net_size(in_dim, 4) + 64;
}

__device__ inline TD3Scratch scratch_at(float* p, int in_dim, int B)
{
    TD3Scratch S;
    S.y = p;
    p += B;
    S.xc = p;
    p += B * kCI;
    S.h1 = p;
    p += B * kH;
    S.h2 = p;
    p += B * kH;
    S.d1 = p;
    p += B * kH;
    S.d2 = p;
    p += B * kH;
    S.d3 = p;
    p += B;
    S.ah1 = p;
    p += B * kH;
    S.ah2 = p;
    p += B * kH;
    S.aout = p;
    p += B * 4;
    S.ad1 = p;
    p += B * kH;
    S.ad2 = p;
    p += B * kH;
    S.ad3 = p;
    p += B * 4;
    S.gq1 = p;
    p += net_size(kCI, 1);
    S.gq2 = p;
    p += net_size(kCI, 1);
    S.ga = p;
    return S;
}

__global__ void __launch_bounds__(kT, 1) td3_update_kernel(TD3Dev A)
{
    extern __shared__ float xs[];  // [B][in_dim] input rows of the current phase
    __shared__ float red[kT / 32];
    const int ag = blockIdx.x, B = A.B, I = A.in_dim, s = threadIdx.x;
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
    TD3Scratch S = scratch_at(A.scratch + (int64_t)ag * A.scratch_floats, I, B);
    const int64_t rb = (int64_t)ag * B + s;  // this sample's row in the [A][B][...] batch arrays
    float h1[kH], h2[kH], x[kCI];

    // ---- 1. target: a' = clip(pi'(o_a') + clip(sigma eps, -c, c), -1, 1); y = r + g (1-d) min Q'
    if (act) {
        float* row = xs + s * I;
        for (int i = 0; i < I; ++i) row[i] = A.o_a2[rb * I + i];
        float at[4];
        fwd(actor_t, row, h1, h2, at, true);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float nz = fminf(fmaxf(A.sigma_t * A.eps[rb * 4 + k], -A.clip_t), A.clip_t);
            at[k] = fminf(fmaxf(at[k] + nz, -1.0f), 1.0f);
        }
        for (int k = 0; k < 28; ++k) x[k] = A.o_c2[rb * 28 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[28 + k] = at[k];
        float q1, q2;
        fwd(Qt[0], x, h1, h2, &q1, false);
        fwd(Qt[1], x, h1, h2, &q2, false);
        S.y[s] = A.r[rb] + A.gamma * (1.0f - A.done[rb]) * fminf(q1, q2);
        // the critic input (o_c, a) of this sample, shared by both critics
        for (int k = 0; k < 28; ++k) S.xc[s * kCI + k] = A.o_c[rb * 28 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) S.xc[s * kCI + 28 + k] = A.a[rb * 4 + k];
    }
    __syncthreads();

    // ---- 2. critics: MSE to y, Adam
    const AdamC Ac{A.lr_critic, A.beta1, A.beta2, A.c1_critic, A.c2_critic, A.adam_eps};
    for (int c = 0; c < 2; ++c) {
        float lossc = 0.0f;
        if (act) {
            float q, d2[kH], d1[kH];
            fwd(Q[c], S.xc + s * kCI, h1, h2, &q, false);
            const float e = q - S.y[s];
            lossc = e * e / (float)B;
            const float dq = 2.0f * e / (float)B;
            bwd_deltas(Q[c], h1, h2, &dq, d2, d1, nullptr);
            for (int j = 0; j < kH; ++j) {
                S.h1[s * kH + j] = h1[j];
                S.h2[s * kH + j] = h2[j];
                S.d1[s * kH + j] = d1[j];
                S.d2[s * kH + j] = d2[j];
            }
            S.d3[s] = dq;
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
        __syncthreads();
    }
    if (!A.update_actor) {
        if (threadIdx.x == 0) A.losses[ag * 3 + 2] = 0.0f;
        return;
    }

    // ---- 3. actor: ascend Q1(o_c, pi(o_a)) through the updated Q1's action input, Adam
    float lossa = 0.0f;
    if (act) {
        float* row = xs + s * I;
        for (int i = 0; i < I; ++i) row[i] = A.o_a[rb * I + i];
        float ah1[kH], ah2[kH], ap[4];
        fwd(actor, row, ah1, ah2, ap, true);
        for (int k = 0; k < 28; ++k) x[k] = S.xc[s * kCI + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[28 + k] = ap[k];
        float q;
        fwd(Q[0], x, h1, h2, &q, false);
        lossa = -q / (float)B;
        const float dq = -1.0f / (float)B;
        float d2[kH], d1[kH], dx[kCI];
        bwd_deltas(Q[0], h1, h2, &dq, d2, d1, dx);
        float d3a[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) d3a[k] = dx[28 + k] * (1.0f - ap[k] * ap[k]);
        float e2[kH], e1[kH];
        bwd_deltas(actor, ah1, ah2, d3a, e2, e1, nullptr);
        for (int j = 0; j < kH; ++j) {
            S.ah1[s * kH + j] = ah1[j];
            S.ah2[s * kH + j] = ah2[j];
            S.ad1[s * kH + j] = e1[j];
            S.ad2[s * kH + j] = e2[j];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) S.ad3[s * 4 + k] = d3a[k];
    }
    const float loss = block_sum(lossa, red);
    if (threadIdx.x == 0) A.losses[ag * 3 + 2] = loss;
    __syncthreads();
    NetP ga = net_at(S.ga, I, 4);
    grad_layer(S.ad1, kH, xs, I, B, kH, I, ga.W1, ga.b1);
    grad_layer(S.ad2, kH, S.ah1, kH, B, kH, kH, ga.W2, ga.b2);
    grad_layer(S.ad3, 4, S.ah2, kH, B, 4, kH, ga.W3, ga.b3);
    __syncthreads();
    const AdamC Aa{A.lr_actor, A.beta1, A.beta2, A.c1_actor, A.c2_actor, A.adam_eps};
    adam(actor.W1, m_a, v_a, S.ga, na, Aa);
    __syncthreads();
    // ---- 4. Polyak averaging of the three targets
    const float tau = A.tau;
    for (int k = threadIdx.x; k < na; k += blockDim.x) actor_t.W1[k] = fmaf(tau, actor.W1[k], (1.0f - tau) * actor_t.W1[k]);
    for (int c = 0; c < 2; ++c)
        for (int k = threadIdx.x; k < nc; k += blockDim.x) Qt[c].W1[k] = fmaf(tau, Q[c].W1[k], (1.0f - tau) * Qt[c].W1[k]);
}

int64_t td3_block_floats(int in_dim) { return 4 * (int64_t)net_size(in_dim, 4) + 8 * (int64_t)net_size(kCI, 1); }
int64_t td3_scratch_bytes(int in_dim, int B) { return 4 * td3_scratch_floats(in_dim, B); }

cudaError_t launch_td3_update(const TD3Dev& A, cudaStream_t s)
{
    if (A.B < 1 || A.B > kT || A.in_dim < 1 || A.in_dim > 256) return cudaErrorNotSupported;
    const size_t smem = (size_t)A.B * A.in_dim * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(td3_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    td3_update_kernel<<<A.n_agents, kT, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace l2f
