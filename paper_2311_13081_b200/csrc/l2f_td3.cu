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
// to a multiple of 4 floats), the actor input rows too.  Two adjacent threads (lanes 2s,
// 2s + 1) own sample s: each computes one half (32) of every hidden layer's outputs from the
// full input vector, which the pair exchanges with warp shuffles; backward deltas are formed as
// partial sums over the thread's half and pair-summed.  So every thread needs at most ~128
// registers and a CTA runs 512 threads (16 warps) -- twice the latency hiding of one thread
// per sample.  Per-sample rows the weight gradients need go to a per-agent global scratch
// (L2-resident).
#include <cmath>
#include <cstdio>

#include <cuda_fp16.h>

#include "l2f_internal.h"

namespace l2f {
namespace {

constexpr int kB = 256;   // max batch
constexpr int kT = 2 * kB;  // two threads per sample
constexpr int kHH = 32;   // half of the hidden width
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

// Rows 32..63 of the staged W1 and W2 sit 4 floats further ("skew"), so the two threads of a
// pair -- reading row j and row j + 32 at the same time -- hit different shared-memory banks.
constexpr int kSkew = 4;

// Debug build only (-DL2F_TD3_TIMING): CTA-0 thread-0 clock() at phase boundaries, printed.
#ifdef L2F_TD3_TIMING
#define TD3_MARK(k)                                              \
    do {                                                         \
        __syncthreads();                                         \
        if (blockIdx.x == 0 && threadIdx.x == 0) mark[k] = clock64(); \
    } while (0)
#else
#define TD3_MARK(k) \
    do {            \
    } while (0)
#endif

__host__ __device__ constexpr int stage_floats(int in, int out)
{
    return kH * pad4(in) + kSkew + kH + kH * kH + kSkew + kH + out * kH + 4;
}

// CTA-cooperative copy of a net into shared memory at sm (16-byte aligned); caller syncs.
__device__ NetS stage(const NetP& n, float* sm)
{
    NetS S;
    S.in = n.in;
    S.out = n.out;
    S.ld1 = pad4(n.in);
    S.W1 = sm;
    S.b1 = S.W1 + kH * S.ld1 + kSkew;
    S.W2 = S.b1 + kH;
    S.b2 = S.W2 + kH * kH + kSkew;
    S.W3 = S.b2 + kH;
    S.b3 = S.W3 + n.out * kH;
    // All loads of a batch are issued before its stores (the global source may not alias the
    // shared destination, but the compiler cannot prove it): 8 loads in flight per thread.
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j0 = threadIdx.x >> 5; j0 < kH; j0 += 2 * nw) {  // a warp per row, two rows at a time
        for (int i0 = lane; i0 < S.ld1; i0 += 128) {
            float t[2][4];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + r * nw, i = i0 + 32 * u;
                    t[r][u] = (j < kH && i < n.in) ? __ldg(n.W1 + j * n.in + i) : 0.0f;
                }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + r * nw, i = i0 + 32 * u;
                    if (j < kH && i < S.ld1) S.W1[j * S.ld1 + (j >= kHH ? kSkew : 0) + i] = t[r][u];
                }
        }
    }
    for (int e0 = threadIdx.x; e0 < kH * kH; e0 += 8 * blockDim.x) {
        float t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            t[u] = e < kH * kH ? __ldg(n.W2 + e) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < kH * kH) S.W2[e + (e >= kHH * kH ? kSkew : 0)] = t[u];
        }
    }
    for (int e = threadIdx.x; e < n.out * kH; e += blockDim.x) S.W3[e] = n.W3[e];
    for (int e = threadIdx.x; e < kH; e += blockDim.x) {
        S.b1[e] = n.b1[e];
        S.b2[e] = n.b2[e];
    }
    if ((int)threadIdx.x < n.out) S.b3[threadIdx.x] = n.b3[threadIdx.x];
    return S;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Input rows [B][I] (global) -> shared [B][LI] zero-padded, a warp per row (coalesced, no
// per-element division).
__device__ __forceinline__ void stage_rows(const float* src, int B, int I, int LI, float* dst)
{
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r0 = threadIdx.x >> 5; r0 < B; r0 += 2 * nw) {  // two rows x 4 chunks per batch
        for (int i0 = lane; i0 < LI; i0 += 128) {
            float t[2][4];
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = r0 + q * nw, i = i0 + 32 * u;
                    t[q][u] = (r < B && i < I) ? __ldg(src + (int64_t)r * I + i) : 0.0f;
                }
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = r0 + q * nw, i = i0 + 32 * u;
                    if (r < B && i < LI) dst[r * LI + i] = t[q][u];
                }
        }
    }
}

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

// ---- half-layer helpers: thread hf in {0, 1} of a sample's pair owns outputs 32 hf .. 32 hf + 31

// out = relu(W1 x + b1) for my 32 outputs, x a shared-memory row of S.ld1 floats (zero padded);
// 16 outputs per pass over the row.
__device__ __forceinline__ void l1_smem_half(const NetS& S, const float* x, int hf, float (&out)[kHH])
{
    const float* Wm = S.W1 + kHH * hf * S.ld1 + kSkew * hf;
    const float* bm = S.b1 + kHH * hf;
#pragma unroll
    for (int jb = 0; jb < kHH; jb += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = bm[jb + j];
#pragma unroll 1
        for (int c = 0; c < S.ld1; c += 4) {
            const float4 xv = ld4(x + c);
#pragma unroll
            for (int j = 0; j < 16; ++j) fma4(acc[j], ld4(Wm + (jb + j) * S.ld1 + c), xv);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[jb + j] = fmaxf(acc[j], 0.0f);
    }
}

// out = relu(W1 x + b1) for my 32 outputs, x the sample's 32-float critic-input row (scratch).
__device__ __forceinline__ void l1_row_half(const NetS& S, const float* xrow, int hf, float (&out)[kHH])
{
    float x[kCI];
#pragma unroll
    for (int c = 0; c < kCI; c += 4) {
        const float4 v = ld4(xrow + c);
        x[c] = v.x;
        x[c + 1] = v.y;
        x[c + 2] = v.z;
        x[c + 3] = v.w;
    }
    const float* Wm = S.W1 + kHH * hf * kCI + kSkew * hf;
    const float* bm = S.b1 + kHH * hf;
#pragma unroll
    for (int j = 0; j < kHH; ++j) {
        float acc = bm[j];
#pragma unroll
        for (int c = 0; c < kCI; c += 4)
            fma4(acc, ld4(Wm + j * kCI + c), make_float4(x[c], x[c + 1], x[c + 2], x[c + 3]));
        out[j] = fmaxf(acc, 0.0f);
        if (j % 8 == 7) sched_fence();
    }
}

// The full 64-vector of a pair from the two halves: lo = outputs 0..31, hi = 32..63.
__device__ __forceinline__ void gather(const float (&mine)[kHH], int hf, float (&lo)[kHH], float (&hi)[kHH])
{
#pragma unroll
    for (int j = 0; j < kHH; ++j) {
        const float o = __shfl_xor_sync(0xffffffffu, mine[j], 1);
        lo[j] = hf ? o : mine[j];
        hi[j] = hf ? mine[j] : o;
    }
}

// out = relu(W2 (lo, hi) + b2) for my 32 outputs.
__device__ __forceinline__ void l2_half(const NetS& S, const float (&lo)[kHH], const float (&hi)[kHH], int hf,
                                        float (&out)[kHH])
{
    const float* Wm = S.W2 + kHH * hf * kH + kSkew * hf;
    const float* bm = S.b2 + kHH * hf;
#pragma unroll
    for (int j = 0; j < kHH; ++j) {
        float acc = bm[j];
#pragma unroll
        for (int c = 0; c < kHH; c += 4)
            fma4(acc, ld4(Wm + j * kH + c), make_float4(lo[c], lo[c + 1], lo[c + 2], lo[c + 3]));
#pragma unroll
        for (int c = 0; c < kHH; c += 4)
            fma4(acc, ld4(Wm + j * kH + kHH + c), make_float4(hi[c], hi[c + 1], hi[c + 2], hi[c + 3]));
        out[j] = fmaxf(acc, 0.0f);
        if (j % 4 == 3) sched_fence();
    }
}

// y = W3 (lo, hi) + b3, all OUT outputs (both threads of the pair), tanh optional.
template <int OUT>
__device__ __forceinline__ void l3_full(const NetS& S, const float (&lo)[kHH], const float (&hi)[kHH], float (&y)[OUT],
                                        bool tanh_out)
{
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
        float acc = S.b3[o];
#pragma unroll
        for (int c = 0; c < kHH; c += 4)
            fma4(acc, ld4(S.W3 + o * kH + c), make_float4(lo[c], lo[c + 1], lo[c + 2], lo[c + 3]));
#pragma unroll
        for (int c = 0; c < kHH; c += 4)
            fma4(acc, ld4(S.W3 + o * kH + kHH + c), make_float4(hi[c], hi[c + 1], hi[c + 2], hi[c + 3]));
        y[o] = tanh_out ? tanhf(acc) : acc;
    }
}

// d2 = (W3^T d3) o relu'(h2) for my 32 outputs.
template <int OUT>
__device__ __forceinline__ void d2_half(const NetS& S, const float (&d3)[OUT], const float (&h2m)[kHH], int hf,
                                        float (&d2m)[kHH])
{
#pragma unroll
    for (int j = 0; j < kHH; ++j) {
        float acc = 0.0f;
#pragma unroll
        for (int o = 0; o < OUT; ++o) acc = fmaf(S.W3[o * kH + kHH * hf + j], d3[o], acc);
        d2m[j] = h2m[j] > 0.0f ? acc : 0.0f;
    }
}

// d1 = (W2^T d2) o relu'(h1), my 32 entries, in place of h1 (h1d1m: h1 in, d1 out): partial
// sums over my 32 rows of W2 for each half of the 64 outputs, pair-summed with one shuffle per
// entry (the partner's partial of my half).
__device__ __forceinline__ void d1_half(const NetS& S, const float (&d2m)[kHH], int hf, float (&h1d1m)[kHH])
{
    const float* Wm = S.W2 + kHH * hf * kH + kSkew * hf;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        float acc[kHH];
#pragma unroll
        for (int i = 0; i < kHH; ++i) acc[i] = 0.0f;
#pragma unroll
        for (int j = 0; j < kHH; ++j) {
#pragma unroll
            for (int c = 0; c < kHH; c += 4) {
                const float4 w = ld4(Wm + j * kH + kHH * half + c);
                acc[c] = fmaf(w.x, d2m[j], acc[c]);
                acc[c + 1] = fmaf(w.y, d2m[j], acc[c + 1]);
                acc[c + 2] = fmaf(w.z, d2m[j], acc[c + 2]);
                acc[c + 3] = fmaf(w.w, d2m[j], acc[c + 3]);
            }
            if (j % 8 == 7) sched_fence();
        }
#pragma unroll
        for (int i = 0; i < kHH; ++i) {
            const float other = __shfl_xor_sync(0xffffffffu, acc[i], 1);
            if (half == hf) h1d1m[i] = h1d1m[i] > 0.0f ? acc[i] + other : 0.0f;
        }
    }
}

__device__ __forceinline__ void store_half(float* row, int hf, const float (&v)[kHH])
{
#pragma unroll
    for (int c = 0; c < kHH; c += 4)
        *reinterpret_cast<float4*>(row + kHH * hf + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
}
__device__ __forceinline__ void load_half(const float* row, int hf, float (&v)[kHH])
{
#pragma unroll
    for (int c = 0; c < kHH; c += 4) {
        const float4 x = ld4(row + kHH * hf + c);
        v[c] = x.x;
        v[c + 1] = x.y;
        v[c + 2] = x.z;
        v[c + 3] = x.w;
    }
}

// Weight gradients of a net's three layers, reduced over the batch: gW[j][i] = sum_s D[s][j]
// X[s][i] (gW row stride K, unpadded: the parameter layout), gb[j] = sum_s D[s][j].
// CTA-cooperative over one tile space holding every layer's 4 x 4 output tiles and ceil(N/4)
// bias tiles (so the three layers and the biases run concurrently, one thread per tile).
// Adjacent threads take adjacent tiles of a row block: their X loads of a sample are
// contiguous, their D loads one broadcast.  D rows (ldd) and X rows (ldx) 16-byte aligned, ldx
// >= pad4(K) with zero padding; N % 4 == 0 or N == 1.
struct GradL {
    const float* D;
    const float* X;
    float *gW, *gb;
    int ldd, ldx, N, K;
};

__device__ void grad_layers(const GradL (&L)[3], int B)
{
    int cnt[3], tot = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const int tj = (L[l].N + 3) / 4, ti = (L[l].K + 3) / 4;
        cnt[l] = tj * ti + tj;
        tot += cnt[l];
    }
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int l = t < cnt[0] ? 0 : (t < cnt[0] + cnt[1] ? 1 : 2);
        const int tile = t - (l > 0 ? cnt[0] : 0) - (l > 1 ? cnt[1] : 0);
        const GradL G = L[l];
        const int ti = (G.K + 3) / 4, nw = ((G.N + 3) / 4) * ti;
        float acc[4][4] = {};
        if (tile < nw) {
            const int j0 = (tile / ti) * 4, i0 = (tile % ti) * 4;
            if (G.N % 4 == 0) {
#pragma unroll 8
                for (int s = 0; s < B; ++s) {
                    const float4 d = ld4(G.D + s * G.ldd + j0), x = ld4(G.X + s * G.ldx + i0);
                    const float dv[4] = {d.x, d.y, d.z, d.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(dv[a], xv[b], acc[a][b]);
                }
            } else {  // N = 1 (the critic's output layer)
#pragma unroll 8
                for (int s = 0; s < B; ++s) {
                    const float d = G.D[s * G.ldd];
                    const float4 x = ld4(G.X + s * G.ldx + i0);
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
                    if (j0 + a < G.N && i0 + b < G.K) G.gW[(j0 + a) * G.K + i0 + b] = acc[a][b];
        } else {  // bias tile: row sums of D
            const int j0 = (tile - nw) * 4;
            if (G.N % 4 == 0) {
#pragma unroll 8
                for (int s = 0; s < B; ++s) {
                    const float4 d = ld4(G.D + s * G.ldd + j0);
                    acc[0][0] += d.x;
                    acc[1][0] += d.y;
                    acc[2][0] += d.z;
                    acc[3][0] += d.w;
                }
            } else {
#pragma unroll 8
                for (int s = 0; s < B; ++s) acc[0][0] += G.D[s * G.ldd];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
                if (j0 + a < G.N) G.gb[j0 + a] = acc[a][0];
        }
    }
}

struct AdamC {
    float lr, b1, b2, c1, c2, eps;  // c1 = 1 - beta1^t, c2 = 1 - beta2^t
};

// Adam on n parameters; with tgt != nullptr also the Polyak step of the matching target net,
// tgt <- tau theta_new + (1 - tau) tgt (the same arithmetic as a separate pass after Adam).
// Four elements per thread per batch, all loads issued before the stores.
__device__ void adam(float* th, float* m, float* v, const float* g, int n, const AdamC& A, float* tgt, float tau)
{
    const int T = blockDim.x;
    for (int k0 = threadIdx.x; k0 < n; k0 += 4 * T) {
        float gk[4], mk[4], vk[4], tk[4], pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + u * T;
            const bool in = k < n;
            gk[u] = in ? g[k] : 0.0f;
            mk[u] = in ? m[k] : 0.0f;
            vk[u] = in ? v[k] : 0.0f;
            tk[u] = in ? th[k] : 0.0f;
            pk[u] = (in && tgt) ? tgt[k] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + u * T;
            if (k < n) {
                const float mn = fmaf(A.b1, mk[u], (1.0f - A.b1) * gk[u]);
                const float vn = fmaf(A.b2, vk[u], (1.0f - A.b2) * gk[u] * gk[u]);
                const float tn = tk[u] - A.lr * (mn / A.c1) / (sqrtf(vn / A.c2) + A.eps);
                m[k] = mn;
                v[k] = vn;
                th[k] = tn;
                if (tgt) tgt[k] = fmaf(tau, tn, (1.0f - tau) * pk[u]);
            }
        }
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
    const int ag = blockIdx.x, B = A.B, I = A.in_dim, LI = pad4(A.in_dim);
    const int s = threadIdx.x >> 1, hf = threadIdx.x & 1;  // sample, half of the pair
    const bool act = s < B;                                // (inactive pairs still shuffle)
    const bool lead = act && hf == 0;                      // writes the per-sample scalars
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
    const int sc = act ? s : 0;  // clamped sample index for inactive lanes' (discarded) loads
    const int64_t rb = (int64_t)ag * B + sc;
    // shared memory: input rows xs [B][LI], then one staged net
    float* xs = sm;
    float* wsm = sm + pad4(B * LI);
    float h1m[kHH], h2m[kHH], lo[kHH], hi[kHH];
    float* const xt = S.d1 + sc * kH;  // target-critic input row (o_c', a'): S.d1 is free until phase 2
    float* const xcr = S.xc + sc * kCI;  // critic input row (o_c, a)

#ifdef L2F_TD3_TIMING
    long long mark[16] = {};
#endif
    TD3_MARK(0);
    // ---- 1. target: a' = clip(pi'(o_a') + clip(sigma eps, -c, c), -1, 1); y = r + g (1-d) min Q'
    stage_rows(A.o_a2 + (int64_t)ag * B * I, B, I, LI, xs);
    NetS W = stage(actor_t, wsm);
    __syncthreads();
    TD3_MARK(12);
    {
        float at[4];
        l1_smem_half(W, xs + sc * LI, hf, h1m);
        gather(h1m, hf, lo, hi);
        l2_half(W, lo, hi, hf, h2m);
        gather(h2m, hf, lo, hi);
        l3_full<4>(W, lo, hi, at, true);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float nz = fminf(fmaxf(A.sigma_t * A.eps[rb * 4 + k], -A.clip_t), A.clip_t);
            at[k] = fminf(fmaxf(at[k] + nz, -1.0f), 1.0f);
        }
        // the pair writes the target-critic input row: lane hf the 16 floats [16 hf, 16 hf + 16)
        if (act) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int q = 16 * hf + k;
                xt[q] = q < 28 ? A.o_c2[rb * 28 + q] : at[q - 28];
            }
        }
    }
    __syncwarp();
    TD3_MARK(13);
    float qmin = 0.0f;
    for (int c = 0; c < 2; ++c) {
        __syncthreads();
        W = stage(Qt[c], wsm);
        __syncthreads();
        float q[1];
        l1_row_half(W, xt, hf, h1m);
        gather(h1m, hf, lo, hi);
        l2_half(W, lo, hi, hf, h2m);
        gather(h2m, hf, lo, hi);
        l3_full<1>(W, lo, hi, q, false);
        qmin = c == 0 ? q[0] : fminf(qmin, q[0]);
    }
    const float y = A.r[rb] + A.gamma * (1.0f - A.done[rb]) * qmin;
    // the critic input row (o_c, a), shared by both critics
    if (act) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int q = 16 * hf + k;
            xcr[q] = q < 28 ? A.o_c[rb * 28 + q] : A.a[rb * 4 + (q - 28)];
        }
    }
    __syncwarp();

    TD3_MARK(1);
    // ---- 2. critics: MSE to y, Adam
    const AdamC Ac{A.lr_critic, A.beta1, A.beta2, A.c1_critic, A.c2_critic, A.adam_eps};
    for (int c = 0; c < 2; ++c) {
        __syncthreads();
        W = stage(Q[c], wsm);
        __syncthreads();
        float q[1], d2m[kHH];
        l1_row_half(W, xcr, hf, h1m);
        if (act) store_half(S.h1 + s * kH, hf, h1m);
        gather(h1m, hf, lo, hi);
        l2_half(W, lo, hi, hf, h2m);
        if (act) store_half(S.h2 + s * kH, hf, h2m);
        gather(h2m, hf, lo, hi);
        l3_full<1>(W, lo, hi, q, false);
        const float e = q[0] - y;
        const float d3[1] = {2.0f * e / (float)B};
        d2_half<1>(W, d3, h2m, hf, d2m);
        if (act) store_half(S.d2 + s * kH, hf, d2m);
        load_half(S.h1 + sc * kH, hf, h1m);  // (reloaded: not kept live across layer 2)
        d1_half(W, d2m, hf, h1m);  // h1m <- my half of d1
        if (act) store_half(S.d1 + s * kH, hf, h1m);
        if (lead) S.d3[s] = d3[0];
        const float loss = block_sum(lead ? e * e / (float)B : 0.0f, red);
        if (threadIdx.x == 0) A.losses[ag * 3 + c] = loss;
        __syncthreads();
        float* g = c == 0 ? S.gq1 : S.gq2;
        NetP gn = net_at(g, kCI, 1);
        TD3_MARK(2 + 3 * c);
        const GradL gl[3] = {{S.d1, S.xc, gn.W1, gn.b1, kH, kCI, kH, kCI},
                             {S.d2, S.h1, gn.W2, gn.b2, kH, kH, kH, kH},
                             {S.d3, S.h2, gn.W3, gn.b3, 1, kH, 1, kH}};
        grad_layers(gl, B);
        __syncthreads();
        TD3_MARK(3 + 3 * c);
        adam(Q[c].W1, m_c[c], v_c[c], g, nc, Ac, A.update_actor ? Qt[c].W1 : nullptr, A.tau);  // (+ Polyak)
        TD3_MARK(4 + 3 * c);
    }
    if (!A.update_actor) {
        if (threadIdx.x == 0) A.losses[ag * 3 + 2] = 0.0f;
        return;
    }

    // ---- 3. actor: ascend Q1(o_c, pi(o_a)) through the updated Q1's action input, Adam
    __syncthreads();
    stage_rows(A.o_a + (int64_t)ag * B * I, B, I, LI, xs);
    W = stage(actor, wsm);
    __syncthreads();
    TD3_MARK(14);
    float ap[4];
    l1_smem_half(W, xs + sc * LI, hf, h1m);
    if (act) store_half(S.ah1 + s * kH, hf, h1m);
    gather(h1m, hf, lo, hi);
    l2_half(W, lo, hi, hf, h2m);
    if (act) store_half(S.ah2 + s * kH, hf, h2m);
    gather(h2m, hf, lo, hi);
    l3_full<4>(W, lo, hi, ap, true);
    if (act && hf == 1) *reinterpret_cast<float4*>(xcr + 28) = make_float4(ap[0], ap[1], ap[2], ap[3]);  // (o_c, pi(o_a))
    TD3_MARK(15);
    __syncthreads();
    W = stage(Q[0], wsm);  // the updated Q1
    __syncthreads();
    float da[4] = {0.f, 0.f, 0.f, 0.f};
    float lossa;
    {
        float q[1], d2m[kHH];
        l1_row_half(W, xcr, hf, h1m);
        if (act) store_half(S.h1 + s * kH, hf, h1m);
        gather(h1m, hf, lo, hi);
        l2_half(W, lo, hi, hf, h2m);
        gather(h2m, hf, lo, hi);
        l3_full<1>(W, lo, hi, q, false);
        lossa = lead ? -q[0] / (float)B : 0.0f;
        const float d3[1] = {-1.0f / (float)B};
        d2_half<1>(W, d3, h2m, hf, d2m);
        load_half(S.h1 + sc * kH, hf, h1m);
        d1_half(W, d2m, hf, h1m);  // h1m <- my half of Q1's d1
        // dL/da = (W1^T d1)[28..31]: partial over my 32 rows of W1, pair-summed
        const float* Wm = W.W1 + kHH * hf * kCI + kSkew * hf;
#pragma unroll
        for (int j = 0; j < kHH; ++j) {
            const float4 w = ld4(Wm + j * kCI + 28);
            da[0] = fmaf(w.x, h1m[j], da[0]);
            da[1] = fmaf(w.y, h1m[j], da[1]);
            da[2] = fmaf(w.z, h1m[j], da[2]);
            da[3] = fmaf(w.w, h1m[j], da[3]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) da[k] += __shfl_xor_sync(0xffffffffu, da[k], 1);
    }
    __syncthreads();
    W = stage(actor, wsm);
    __syncthreads();
    {
        float d3a[4], e2m[kHH];
#pragma unroll
        for (int k = 0; k < 4; ++k) d3a[k] = da[k] * (1.0f - ap[k] * ap[k]);
        load_half(S.ah2 + sc * kH, hf, h2m);
        d2_half<4>(W, d3a, h2m, hf, e2m);
        if (act) store_half(S.ad2 + s * kH, hf, e2m);
        load_half(S.ah1 + sc * kH, hf, h1m);
        d1_half(W, e2m, hf, h1m);  // h1m <- my half of the actor's d1
        if (act) store_half(S.ad1 + s * kH, hf, h1m);
        if (lead) *reinterpret_cast<float4*>(S.ad3 + s * 4) = make_float4(d3a[0], d3a[1], d3a[2], d3a[3]);
    }
    const float loss = block_sum(lossa, red);
    if (threadIdx.x == 0) A.losses[ag * 3 + 2] = loss;
    __syncthreads();
    NetP ga = net_at(S.ga, I, 4);
    TD3_MARK(8);
    const GradL gl[3] = {{S.ad1, xs, ga.W1, ga.b1, kH, LI, kH, I},
                         {S.ad2, S.ah1, ga.W2, ga.b2, kH, kH, kH, kH},
                         {S.ad3, S.ah2, ga.W3, ga.b3, 4, kH, 4, kH}};
    grad_layers(gl, B);
    __syncthreads();
    const AdamC Aa{A.lr_actor, A.beta1, A.beta2, A.c1_actor, A.c2_actor, A.adam_eps};
    TD3_MARK(9);
    adam(actor.W1, m_a, v_a, S.ga, na, Aa, actor_t.W1, A.tau);  // ---- 4. with the actor target's Polyak step
    TD3_MARK(10);
    TD3_MARK(11);
#ifdef L2F_TD3_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        printf("L2F_TD3 target %lld critic0 fwdbwd %lld grads %lld adam %lld critic1 fwdbwd %lld grads %lld adam %lld "
               "actor fwdbwd %lld grads %lld adam %lld polyak %lld total %lld\n",
               mark[1] - mark[0], mark[2] - mark[1], mark[3] - mark[2], mark[4] - mark[3], mark[5] - mark[4],
               mark[6] - mark[5], mark[7] - mark[6], mark[8] - mark[7], mark[9] - mark[8], mark[10] - mark[9],
               mark[11] - mark[10], mark[11] - mark[0]);
        printf("L2F_TD3 target: stage %lld actor fwd %lld critics %lld; actor: stage %lld fwd %lld rest %lld\n",
               mark[12] - mark[0], mark[13] - mark[12], mark[1] - mark[13], mark[14] - mark[7], mark[15] - mark[14],
               mark[8] - mark[15]);
    }
#endif
}

size_t td3_smem_bytes(int in_dim, int B)
{
    const int a = stage_floats(in_dim, 4), c = stage_floats(kCI, 1);
    return (size_t)(pad4(B * pad4(in_dim)) + (a > c ? a : c)) * sizeof(float);
}

}  // namespace

__global__ void td3_export_actor_kernel(const float* __restrict__ actor, int n, uint16_t* __restrict__ out)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        out[k] = __half_as_ushort(__float2half_rn(actor[k]));
}

cudaError_t launch_td3_export_actor(const float* params, int64_t block, int agent, int in_dim, uint16_t* out,
                                    cudaStream_t s)
{
    const int n = net_size(in_dim, 4);
    td3_export_actor_kernel<<<(n + 255) / 256, 256, 0, s>>>(params + (int64_t)agent * block, n, out);
    return cudaGetLastError();
}

int64_t td3_block_floats(int in_dim) { return 4 * (int64_t)net_size(in_dim, 4) + 8 * (int64_t)net_size(kCI, 1); }
int64_t td3_scratch_bytes(int in_dim, int B) { return 4 * td3_scratch_floats(in_dim, B); }

cudaError_t launch_td3_update(const TD3Dev& A, cudaStream_t s)
{
    if (A.B < 1 || A.B > kB || A.in_dim < 1 || A.in_dim > 256) return cudaErrorNotSupported;
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
