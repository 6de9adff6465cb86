// l2f_td3.cu -- GPU-batched TD3 update ("we use TD3", S:368-455;
// DESIGN.md Q32-Q35), sm_100a.
//
// One CTA (512 threads) per agent: many independent agents (seeds, ablation configurations --
// the paper's Table II runs 10 configurations x 50 seeds) are updated concurrently, one per SM.
// FP32 master weights in a flat per-agent block:
//   [actor, actor', Q1, Q2, Q1', Q2', m_actor, v_actor, m_Q1, v_Q1, m_Q2, v_Q2]
// each net W1[hid][in], b1, W2[hid][hid], b2, W3[out][hid], b3 (the oracle's layout; the actor
// part is the l2f_policy layout, so it exports to the tcgen05 rollout after fp16 rounding).
//
// Per update: (1) target actions with clipped smoothing noise and the clipped double-Q target
// y; (2) per critic: forward, per-sample deltas, weight gradients as D^T X reductions over
// the batch, Adam (+ the target's Polyak step on delayed updates); (3) on delayed steps the
// deterministic policy gradient through the updated Q1's action input, Adam + Polyak.
//
// Every hidden layer is a CTA-wide batch GEMM with the activations in shared memory: the
// batch's rows of one layer ([256][64] FP32, 64 KB, float4 slots XOR-swizzled by row so four
// consecutive rows read the same column from four different banks), the critic input rows
// ([256][32]), and the net in use (rows padded to an odd number of float4s, so eight
// consecutive weight rows start in eight different bank groups).  A thread owns a 4-sample x
// 8-output register tile: per 4-input chunk it loads 4 activation float4s and 8 weight float4s
// for 128 FMAs (the thread-per-sample formulation loads a weight float4 per 4 FMAs and is
// shared-memory bound; the pairs feed packed FFMA2).  Backward deltas are the same GEMM
// against W2 (in place, masked by ReLU'); weight gradients are 8 x 4 tiles over a warp's
// sample range, the ranges summed into a shared-memory gradient block in fixed order
// (deterministic), which Adam reads.  A warp owns the rows of its 16 samples in every
// per-sample step, so those steps need only warp barriers.  Nets and the actor input rows
// (in_dim floats, the one operand that does not fit) are staged by cp.async, the input rows
// in column parts into whichever activation buffers are free at that point.
#include <cmath>
#include <cstdio>

#include <cuda_fp16.h>

#include "l2f_internal.h"

namespace l2f {
namespace {

constexpr int kB = 256;     // max batch = rows of the activation buffers
constexpr int kT = 512;     // threads per CTA
constexpr int kH = 64;      // hidden width
constexpr int kCI = 32;     // critic input: o_c (28) + a (4)
constexpr int kMaxIn = 156; // actor input bound (shared-memory plan)
constexpr int kLd2 = 68;    // staged W2 row stride (17 float4s)

#ifndef L2F_TD3_UNROLL
#define L2F_TD3_UNROLL 1  // unroll of the GEMM chunk loops (1: 6.23e5, 2: 6.09e5, 4: 5.84e5 updates/s; spills grow)
#endif
#ifndef L2F_TD3_UNROLL_BWD
#define L2F_TD3_UNROLL_BWD L2F_TD3_UNROLL
#endif
#ifndef L2F_TD3_UNROLL_WG
#define L2F_TD3_UNROLL_WG 2  // the weight-gradient sample loop (4 samples per trip)
#endif
#define L2F_TD3_STR(x) #x
#define L2F_TD3_PRAGMA(x) _Pragma(L2F_TD3_STR(x))
#define L2F_TD3_PRAGMA_UNROLL L2F_TD3_PRAGMA(unroll L2F_TD3_UNROLL)

__host__ __device__ constexpr int net_size(int in, int out) { return kH * in + kH + kH * kH + kH + out * kH + out; }
__host__ __device__ constexpr int pad4(int k) { return (k + 3) & ~3; }
// Staged W1 row stride: a multiple of 4 floats with an odd float4 count.
__host__ __device__ constexpr int ldw_of(int in) { return ((pad4(in) / 4) & 1) ? pad4(in) : pad4(in) + 4; }
__host__ __device__ constexpr int stage_floats(int in, int out)
{
    return kH * ldw_of(in) + kH + kH * kLd2 + kH + out * kH + 4;
}

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

struct NetS {  // a net staged in shared memory
    const float *W1, *b1, *W2, *b2, *W3, *b3;
    int ld1;
};

// Debug build only (-DL2F_TD3_TIMING): CTA-0 thread-0 clock() at phase boundaries, printed.
#ifdef L2F_TD3_TIMING
#define TD3_MARK(k)                                                  \
    do {                                                             \
        __syncthreads();                                             \
        if (blockIdx.x == 0 && threadIdx.x == 0) mark[k] = clock64(); \
    } while (0)
__device__ long long g_td3_sub[32];
#define TD3_SUB(k)                                                          \
    do {                                                                    \
        __syncthreads();                                                    \
        if (blockIdx.x == 0 && threadIdx.x == 0) g_td3_sub[k] = clock64(); \
    } while (0)
#else
#define TD3_MARK(k) \
    do {            \
    } while (0)
#define TD3_SUB(k) \
    do {           \
    } while (0)
#endif

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ void fma4(float& acc, float4 w, float4 x)
{
    acc = fmaf(w.x, x.x, acc);
    acc = fmaf(w.y, x.y, acc);
    acc = fmaf(w.z, x.z, acc);
    acc = fmaf(w.w, x.w, acc);
}

// Packed FP32 pairs (FFMA2): acc.x accumulates the even, acc.y the odd input of each pair.
__device__ __forceinline__ void fma4x2(float2& acc, float4 w, float4 x)
{
    acc = __ffma2_rn(make_float2(w.x, w.y), make_float2(x.x, x.y), acc);
    acc = __ffma2_rn(make_float2(w.z, w.w), make_float2(x.z, x.w), acc);
}

__device__ __forceinline__ float comp(float4 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

// Activation buffers: row s of ld floats (ld = 32 or 64), float4 slot c4 stored at slot
// c4 ^ (s & 3): four consecutive rows put the same column in four different bank groups, and
// the rows s0 + 4 i a GEMM thread owns share one key (s0 & 3), so their addresses differ by
// compile-time offsets.
__device__ __forceinline__ int sw(int s, int c4, int ld) { return s * ld + ((c4 ^ (s & 3)) << 2); }
__device__ __forceinline__ float& at(float* buf, int s, int k, int ld) { return buf[sw(s, k >> 2, ld) + (k & 3)]; }

struct XSp {  // a plain shared-memory row buffer (row stride ld floats, 16-byte aligned rows)
    const float* p;
    int ld;
    __device__ __forceinline__ float4 operator()(int s, int c4) const { return ld4(p + s * ld + 4 * c4); }
};

// The actor input is consumed in column parts of up to kPW floats (kPW / 16 = 5 gradient
// column blocks), staged in shared memory rows of kPLd floats (21 float4s: four consecutive
// rows hit four different bank groups).
constexpr int kPW = 80;
constexpr int kPLd = 84;

__device__ __forceinline__ void cp_async(float* dst, const float* src, int bytes_total, int bytes_src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if (bytes_total == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes_src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(bytes_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Columns [k0, k0 + w) of the batch rows X [B][I] (global) -> dst rows of ld floats (plain),
// or, with ld == 0, the swizzled 64-float activation layout (w <= 64), by cp.async (every copy
// in flight at once), zero beyond I; a warp per row.  Caller waits + syncs.
__device__ __forceinline__ int stage_off(int r, int q, int ld)  // float offset of column q of row r
{
    return ld ? r * ld + q : r * kH + ((((q >> 2) ^ (r & 3)) << 2) | (q & 3));
}
__device__ void stage_cols(const float* X, int B, int I, int k0, int w, float* dst, int ld = kPLd)
{
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (!(I & 1)) {  // 8-byte pieces (I even: rows 8-byte aligned; a piece never straddles a slot)
        const int np = (w + 1) >> 1;
        for (int r = threadIdx.x >> 5; r < B; r += nw)
            for (int q = lane; q < np; q += 32) {
                const int k = k0 + 2 * q;
                const int b = k + 2 <= I ? 8 : (k < I ? 4 : 0);
                cp_async(dst + stage_off(r, 2 * q, ld), X + (int64_t)r * I + (b ? k : 0), 8, b);
            }
    } else {
        for (int r = threadIdx.x >> 5; r < B; r += nw)
            for (int q = lane; q < w; q += 32) {
                const int k = k0 + q;
                cp_async(dst + stage_off(r, q, ld), X + (int64_t)r * I + (k < I ? k : 0), 4, k < I ? 4 : 0);
            }
    }
}

// rows x cols (global, row stride gs) -> shared (row stride ds), columns cols..ds-1 zeroed:
// 4-byte cp.async, a warp per row, every copy of the thread in flight at once (the source may
// have been written by this kernel earlier: cp.async reads through L1 like a plain load).
// Caller waits (cp_async_wait_all) and syncs.
__device__ void copy_rows(const float* g, int rows, int cols, int gs, float* d, int ds)
{
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = threadIdx.x >> 5; r < rows; r += nw)
        for (int i = lane; i < ds; i += 32) cp_async(d + r * ds + i, g + (int64_t)r * gs + (i < cols ? i : 0), 4, i < cols ? 4 : 0);
}

// CTA-cooperative copy of a net into shared memory at sm (16-byte aligned): issues the
// copies (stage_issue) or issues and waits for this thread's (stage); caller syncs.
__device__ __forceinline__ NetS stage_view(int in, int out, float* sm)  // where stage_issue puts a net
{
    NetS S;
    S.ld1 = ldw_of(in);
    float* W1 = sm;
    float* b1 = W1 + kH * S.ld1;
    float* W2 = b1 + kH;
    float* b2 = W2 + kH * kLd2;
    float* W3 = b2 + kH;
    S.W1 = W1;
    S.b1 = b1;
    S.W2 = W2;
    S.b2 = b2;
    S.W3 = W3;
    S.b3 = W3 + out * kH;
    return S;
}

__device__ NetS stage_issue(const NetP& n, float* sm)
{
    const NetS S = stage_view(n.in, n.out, sm);
    copy_rows(n.W1, kH, n.in, n.in, const_cast<float*>(S.W1), S.ld1);
    copy_rows(n.W2, kH, kH, kH, const_cast<float*>(S.W2), kLd2);
    copy_rows(n.W3, n.out, kH, kH, const_cast<float*>(S.W3), kH);
    float* b1 = const_cast<float*>(S.b1);
    float* b2 = const_cast<float*>(S.b2);
    float* b3 = const_cast<float*>(S.b3);
    for (int e = threadIdx.x; e < 2 * kH + n.out; e += blockDim.x) {
        const float* src = e < kH ? n.b1 + e : (e < 2 * kH ? n.b2 + (e - kH) : n.b3 + (e - 2 * kH));
        float* dst = e < kH ? b1 + e : (e < 2 * kH ? b2 + (e - kH) : b3 + (e - 2 * kH));
        cp_async(dst, src, 4, 4);
    }
    return S;
}

__device__ NetS stage(const NetP& n, float* sm)
{
    const NetS S = stage_issue(n, sm);
    cp_async_wait_all();  // (the caller's barrier publishes)
    return S;
}

// Warp w reads and writes only the rows [16 w, 16 w + 16) of the activation buffers in every
// per-sample step (forward and delta GEMMs, output layer, critic-input rows): between two such
// steps a warp barrier suffices; the CTA barrier is needed only around the weight-gradient
// reductions (all rows), staging and restaging of the shared net, and the row save/restore.
__device__ __forceinline__ void own_rows_sync() { __syncwarp(); }

// ---- CTA-wide batch GEMMs over the activation rows (no barriers inside) ----

// Y = act(X W^T + b) for a 64-output layer, W rows of stride ldw (K4 float4 chunks, zero
// padded).  Warp w owns samples 16 w .. 16 w + 15; lane (g = lane & 3, o = lane >> 2) the
// samples 16 w + g + 4 i (i < 4) -- four consecutive rows per load instruction -- and the
// outputs o + 8 m (m < 8) -- eight consecutive weight rows per load instruction.
template <class XA>
__device__ __forceinline__ void fwd_acc(const XA& X, int c0, int nc, const float* W, int ldw, float2 (&acc)[4][8])
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 3, o = lane >> 2;
    const int s0 = 16 * w + g;
    const float* Wo = W + o * ldw + 4 * c0;
L2F_TD3_PRAGMA_UNROLL
    for (int c = 0; c < nc; ++c) {
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = X(s0 + 4 * i, c);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float4 wv = ld4(Wo + 8 * m * ldw + 4 * c);
#pragma unroll
            for (int i = 0; i < 4; ++i) fma4x2(acc[i][m], wv, x[i]);
        }
    }
}

__device__ __forceinline__ void fwd_init(const float* b, float2 (&acc)[4][8])
{
    const int o = (threadIdx.x & 31) >> 2;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const float bj = b[o + 8 * m];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][m] = make_float2(bj, 0.0f);
    }
}

__device__ __forceinline__ void fwd_store(const float2 (&acc)[4][8], float* Y, bool relu)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 3, o = lane >> 2;
    const int s0 = 16 * w + g;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float v = acc[i][m].x + acc[i][m].y;
            at(Y, s0 + 4 * i, o + 8 * m, kH) = relu ? fmaxf(v, 0.0f) : v;
        }
}

// Y = relu(X W^T + b) with X a swizzled activation buffer (row ld = 32 or 64 floats): the
// thread's four rows s0 + 4 i share the swizzle key g = s0 & 3, so one XOR per chunk
// addresses all four.
__device__ __forceinline__ void fwd_gemm(const float* X, int ld, const float* W, int ldw, const float* b, float* Y,
                                         int B)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 3, o = lane >> 2;
    if (16 * w >= B) return;
    float2 acc[4][8];
    fwd_init(b, acc);
    const float* xr = X + (16 * w + g) * ld;
    const float* Wo = W + o * ldw;
L2F_TD3_PRAGMA_UNROLL
    for (int c = 0; c < ld / 4; ++c) {
        const float* xc = xr + 4 * (c ^ g);
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = ld4(xc + 4 * i * ld);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float4 wv = ld4(Wo + 8 * m * ldw + 4 * c);
#pragma unroll
            for (int i = 0; i < 4; ++i) fma4x2(acc[i][m], wv, x[i]);
        }
    }
    fwd_store(acc, Y, true);
}

// Chunks [c0, c0 + nc) of the input layer from a swizzled 64-float row buffer (local chunk
// c at slot c ^ g for the thread's four rows).
__device__ __forceinline__ void fwd_acc_sw(const float* X, int c0, int nc, const float* W, int ldw,
                                           float2 (&acc)[4][8])
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 3, o = lane >> 2;
    const float* xr = X + (16 * w + g) * kH;
    const float* Wo = W + o * ldw + 4 * c0;
L2F_TD3_PRAGMA_UNROLL
    for (int c = 0; c < nc; ++c) {
        const float* xc = xr + 4 * (c ^ g);
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = ld4(xc + 4 * i * kH);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float4 wv = ld4(Wo + 8 * m * ldw + 4 * c);
#pragma unroll
            for (int i = 0; i < 4; ++i) fma4x2(acc[i][m], wv, x[i]);
        }
    }
}

// The actor's input layer, Y = relu(X W1^T + b1), X [B][I] global rows (I <= kMaxIn): the
// net (n -> Wsm) and both column parts of X are staged by one wave of cp.async -- columns
// [0, kP0) into rows of kP0 floats at P0buf (B + X32: free here), the rest (<= 64) swizzled
// into Y itself (free until the layer's output is stored, after a barrier).  Contains
// barriers: all threads call it.
constexpr int kP0 = 92;  // 23 float4s (odd: four consecutive rows hit four bank groups)
__device__ void input_rows_issue(const float* X, int I, int B, float* Y, float* P0buf)
{
    const int K4 = pad4(I) / 4, c1 = min(K4, kP0 / 4);
    stage_cols(X, B, I, 0, 4 * c1, P0buf, kP0);
    if (K4 > c1) stage_cols(X, B, I, kP0, 4 * (K4 - c1), Y, 0);
}
__device__ NetS input_issue(const NetP& n, float* Wsm, const float* X, int I, int B, float* Y, float* P0buf)
{
    const NetS W = stage_issue(n, Wsm);
    input_rows_issue(X, I, B, Y, P0buf);
    return W;
}
__device__ void input_compute(const NetS& W, int I, int B, float* Y, float* P0buf)
{
    cp_async_wait_all();
    __syncthreads();
    TD3_SUB(0);
    const int K4 = pad4(I) / 4, c1 = min(K4, kP0 / 4);
    const bool busy = 16 * (int)(threadIdx.x >> 5) < B;
    float2 acc[4][8];
    fwd_init(W.b1, acc);
    if (busy) {
        fwd_acc(XSp{P0buf, kP0}, 0, c1, W.W1, W.ld1, acc);
        if (K4 > c1) fwd_acc_sw(Y, c1, K4 - c1, W.W1, W.ld1, acc);
    }
    own_rows_sync();  // (Y held the second part: the warp's own rows)
    TD3_SUB(1);
    if (busy) fwd_store(acc, Y, true);
}
__device__ NetS fwd_input_layer(const NetP& n, float* Wsm, const float* X, int I, int B, float* Y, float* P0buf)
{
    const NetS W = input_issue(n, Wsm, X, I, B, Y, P0buf);
    input_compute(W, I, B, Y, P0buf);
    return W;
}

// In place: H[s][k] <- (sum_j D[s][j] W2[j][k]) if H[s][k] > 0 else 0 (the delta through a
// ReLU layer), k < 64.  Tile: samples 16 w + g + 4 i, outputs k = 8 o .. 8 o + 7.
__device__ __forceinline__ void bwd_gemm(const float* D, const float* W2, float* H, int B)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 3, o = lane >> 2;
    if (16 * w >= B) return;
    const int s0 = 16 * w + g;
    float2 acc[4][4];  // (k, k + 1) pairs of outputs 8 o + 2 q, FFMA2
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = make_float2(0.0f, 0.0f);
L2F_TD3_PRAGMA(unroll L2F_TD3_UNROLL_BWD)
    for (int c = 0; c < kH / 4; ++c) {
        float4 d[4];
        const float* dc = D + s0 * kH + 4 * (c ^ g);  // (rows s0 + 4 i share the key g)
#pragma unroll
        for (int i = 0; i < 4; ++i) d[i] = ld4(dc + 4 * i * kH);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const float* wr = W2 + (4 * c + jj) * kLd2 + 8 * o;
            const float4 wa = ld4(wr), wb = ld4(wr + 4);
            const float2 wp[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                                  make_float2(wb.z, wb.w)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float dv = comp(d[i], jj);
                const float2 dd = make_float2(dv, dv);
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = __ffma2_rn(dd, wp[q], acc[i][q]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int s = s0 + 4 * i;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            float* p = H + sw(s, 2 * o + hh, kH);
            const float4 h = ld4(p);
            const float2 a = acc[i][2 * hh], b = acc[i][2 * hh + 1];
            st4(p, make_float4(h.x > 0.0f ? a.x : 0.0f, h.y > 0.0f ? a.y : 0.0f, h.z > 0.0f ? b.x : 0.0f,
                               h.w > 0.0f ? b.y : 0.0f));
        }
    }
}

// Partial weight gradients of a 64-output layer over S contiguous sample ranges (one warp
// each per column block): P[p][j][k] = sum_{s in range p} D[s][j] X[s][k] (k < K, row
// stride K), Pb[p][j] = sum D[s][j].  Warp (wc, p) covers k = 16 wc .. 16 wc + 15; lane (jg
// = lane >> 2, kq = lane & 3) the 8 x 4 tile j = 8 jg + a, k = 16 wc + 4 kq + b.  The
// partial ranges are summed by the Adam pass (fixed order).
template <bool SWX>
__device__ __forceinline__ void wgrad(const float* D, const float* X, int ldx, int K, int B, int S, float* P,
                                      float* Pb, int ldP = -1, bool with_bias = true, float* tmp = nullptr,
                                      float* tmpb = nullptr)
{
    if (ldP < 0) ldP = K;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, jg = lane >> 2, kq = lane & 3;
    const int NC = (K + 15) / 16;
    const bool active = w < NC * S;
    const int wc = w % NC, p = active ? w / NC : S;
    const int ch = (((B + S - 1) / S) + 3) & ~3;  // ranges start at multiples of 4: s & 3 = unrolled j
    const int sb = min(B, (active ? p : 0) * ch), se = min(B, sb + ch);
    const int c4 = 4 * wc + kq;
    const bool bias = with_bias && wc == 0 && kq == 0;
    // D rows (swizzled, 64): logical slots 2 jg, 2 jg + 1 of row s sit at (2 jg ^ (s & 2)) + {0, 1},
    // swapped when s is odd; X slot c4 at c4 ^ (s & 3) (swizzled) or c4 (plain)
    int doff[2], xoff[4];
#pragma unroll
    for (int e = 0; e < 2; ++e) doff[e] = ((2 * jg) ^ (2 * e)) << 2;
#pragma unroll
    for (int j = 0; j < 4; ++j) xoff[j] = SWX ? ((c4 ^ j) << 2) : (c4 << 2);
    float2 acc[4][4], bacc[4];  // rows (8 jg + 2 q, 8 jg + 2 q + 1) as FFMA2 pairs
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        bacc[q] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[q][b] = make_float2(0.0f, 0.0f);
    }
    auto body = [&](int s, int j) {  // j = s & 3 (compile-time in the main loop)
        const float* dr = D + s * kH + doff[(j >> 1) & 1];
        const float4 da = ld4(dr + 4 * (j & 1)), db = ld4(dr + 4 * ((j & 1) ^ 1));
        const float4 x = ld4(X + s * ldx + xoff[j & 3]);
        const float2 dp[4] = {make_float2(da.x, da.y), make_float2(da.z, da.w), make_float2(db.x, db.y),
                              make_float2(db.z, db.w)};
        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float2 xx = make_float2(xv[b], xv[b]);
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][b] = __ffma2_rn(dp[q], xx, acc[q][b]);
        }
        if (bias)
#pragma unroll
            for (int q = 0; q < 4; ++q) bacc[q] = __fadd2_rn(bacc[q], dp[q]);
    };
    if (active) {
        const int se4 = sb + ((se - sb) & ~3);
L2F_TD3_PRAGMA(unroll L2F_TD3_UNROLL_WG)
        for (int s4 = sb; s4 < se4; s4 += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) body(s4 + j, j);
        }
        for (int s = se4; s < se; ++s) body(s, s & 3);
    }
    // the S ranges' partial tiles are summed into the shared-memory gradient P (row stride ldP)
    // and Pb in range order (deterministic).  With a free buffer (tmp: S x 64 x K, tmpb: S x 64)
    // every range writes its partial tile at once and one pass sums them after one barrier;
    // otherwise range 0 stores and ranges 1 .. S-1 add, a barrier between.  All threads take
    // part in the barriers.
    if (tmp) {
        if (p < S) {
            float* t0 = tmp + p * kH * K;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (4 * c4 + b < K) {
                        t0[(8 * jg + 2 * q) * K + 4 * c4 + b] = acc[q][b].x;
                        t0[(8 * jg + 2 * q + 1) * K + 4 * c4 + b] = acc[q][b].y;
                    }
            if (bias)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tmpb[p * kH + 8 * jg + 2 * q] = bacc[q].x;
                    tmpb[p * kH + 8 * jg + 2 * q + 1] = bacc[q].y;
                }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kH * K + (with_bias ? kH : 0); e += blockDim.x) {
            const bool wgt = e < kH * K;
            const float* src = wgt ? tmp + e : tmpb + (e - kH * K);
            const int st = wgt ? kH * K : kH;
            float v = src[0];
            for (int r = 1; r < S; ++r) v += src[r * st];
            if (wgt)
                P[(e / K) * ldP + e % K] = v;
            else
                Pb[e - kH * K] = v;
        }
        __syncthreads();
        return;
    }
    for (int r = 0; r < S; ++r) {
        if (p == r) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (4 * c4 + b < K) {
                        float* g0 = P + (8 * jg + 2 * q) * ldP + 4 * c4 + b;
                        float* g1 = g0 + ldP;
                        *g0 = r ? *g0 + acc[q][b].x : acc[q][b].x;
                        *g1 = r ? *g1 + acc[q][b].y : acc[q][b].y;
                    }
            if (bias)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float* b0 = Pb + 8 * jg + 2 * q;
                    b0[0] = r ? b0[0] + bacc[q].x : bacc[q].x;
                    b0[1] = r ? b0[1] + bacc[q].y : bacc[q].y;
                }
        }
        __syncthreads();
    }
}

// Output-layer gradients (out <= 4 outputs) into shared memory: G[o][k] = sum_s d3[s][o]
// H[s][k] (row stride 64) and, contiguous after it, Gb[o] = sum_s d3[s][o]; 8 sample ranges
// (thread t: k = t & 63, range t >> 6) write their partial rows to tmp (8 x (64 out + out)
// floats), one barrier, then one pass sums them in range order (deterministic).  H is no
// longer read after the barrier; G is complete only after the caller's next barrier.
__device__ __forceinline__ void wgrad_out(const float* d3, int out, const float* H, int B, float* G, float* tmp)
{
    const int k = threadIdx.x & 63, p = threadIdx.x >> 6;
    const int ch = (B + 7) / 8, sb = min(B, p * ch), se = min(B, sb + ch);
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, bacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int s = sb; s < se; ++s) {
        const float h = H[sw(s, k >> 2, kH) + (k & 3)];
        const float4 d = ld4(d3 + 4 * s);
        const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            acc[o] = fmaf(dv[o], h, acc[o]);
            bacc[o] += dv[o];
        }
    }
    const int rl = out * kH + out;
    for (int o = 0; o < out; ++o) {
        tmp[p * rl + o * kH + k] = acc[o];
        if (k == 0) tmp[p * rl + out * kH + o] = bacc[o];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rl; e += blockDim.x) {
        float v = tmp[e];
        for (int r = 1; r < 8; ++r) v += tmp[r * rl + e];
        G[e] = v;
    }
}

// Per-sample helpers, thread pair (s, hf): hf = 0/1 handles columns 32 hf .. 32 hf + 31.

// y[o] = b3[o] + W3[o] . H[s], o < OUT (both threads of the pair get all of y).
template <int OUT>
__device__ __forceinline__ void out_layer(const NetS& W, const float* H, int s, int hf, float (&y)[OUT])
{
    float acc[OUT];
#pragma unroll
    for (int o = 0; o < OUT; ++o) acc[o] = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int c4 = 8 * hf + c;
        const float4 h = ld4(H + sw(s, c4, kH));
#pragma unroll
        for (int o = 0; o < OUT; ++o) fma4(acc[o], ld4(W.W3 + o * kH + 4 * c4), h);
    }
#pragma unroll
    for (int o = 0; o < OUT; ++o) y[o] = acc[o] + __shfl_xor_sync(0xffffffffu, acc[o], 1) + W.b3[o];
}

// In place: H[s][j] <- (sum_o W3[o][j] d3[o]) if H[s][j] > 0 else 0, my 32 columns.
template <int OUT>
__device__ __forceinline__ void out_back(const NetS& W, float* H, int s, int hf, const float (&d3)[OUT])
{
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int c4 = 8 * hf + c;
        float* p = H + sw(s, c4, kH);
        const float4 h = ld4(p);
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int o = 0; o < OUT; ++o) {
            const float4 w = ld4(W.W3 + o * kH + 4 * c4);
            r.x = fmaf(w.x, d3[o], r.x);
            r.y = fmaf(w.y, d3[o], r.y);
            r.z = fmaf(w.z, d3[o], r.z);
            r.w = fmaf(w.w, d3[o], r.w);
        }
        st4(p, make_float4(h.x > 0.0f ? r.x : 0.0f, h.y > 0.0f ? r.y : 0.0f, h.z > 0.0f ? r.z : 0.0f,
                           h.w > 0.0f ? r.w : 0.0f));
    }
}

// Critic input row s of X32: (o_c[s] (28), act (4)), this thread's 16 floats.
__device__ __forceinline__ void put_critic_row(float* X32, int s, int hf, const float* oc, const float (&act)[4])
{
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int c4 = 4 * hf + c;
        float4 v;
        if (c4 < 7)
            v = __ldg(reinterpret_cast<const float4*>(oc) + c4);  // (rows of 28 floats: 16-byte aligned)
        else
            v = make_float4(act[0], act[1], act[2], act[3]);
        st4(X32 + sw(s, c4, kCI), v);
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

// Sample ranges of the input layer's weight gradient: the warps not needed for the column
// blocks of one staged part (<= kPW / 16 blocks) split the batch.
__host__ __device__ inline int wg_splits(int in)
{
    const int nc = (in + 15) / 16;
    return 16 / (nc < kPW / 16 ? nc : kPW / 16);
}

// Shared-memory gradient of a net in the parameter layout (W1 [64][in], b1, W2, b2, W3, b3).
struct GradS {
    float *W1, *b1, *W2, *b2, *W3, *b3;
};
__device__ __forceinline__ GradS grad_at(float* p, int in, int out)
{
    GradS G;
    G.W1 = p;
    G.b1 = G.W1 + kH * in;
    G.W2 = G.b1 + kH;
    G.b2 = G.W2 + kH * kH;
    G.W3 = G.b2 + kH;
    G.b3 = G.W3 + out * kH;
    return G;
}

// Backward of a net from its two activation buffers, up to the input layer's delta: Hb =
// H2 (-> D2 in place), Ha = H1 (-> D1 in place); d3 rows (4 floats) in smem.  Writes the
// W3/b3 gradient to G3 and the W2/b2 gradient to G2 (shared memory, parameter layout); the
// caller does W1/b1 (from its input rows).  Ends with a barrier.
__device__ void net_backward(const NetS& W, int out, const float* d3s, float* Ha, float* Hb, int B, int s, int hf,
                             const float (&d3)[4], const GradS& G3, const GradS& G2, float* tmp)
{
    wgrad_out(d3s, out, Hb, B, G3.W3, tmp);  // (G3.b3 follows G3.W3; Hb free after its barrier)
    if (out == 1) {
        const float d1[1] = {d3[0]};
        out_back<1>(W, Hb, s, hf, d1);
    } else {
        out_back<4>(W, Hb, s, hf, d3);
    }
    __syncthreads();
    wgrad<true>(Hb, Ha, kH, kH, B, 4, G2.W2, G2.b2);  // (ends with a barrier)
    bwd_gemm(Hb, W.W2, Ha, B);
    __syncthreads();
}

struct AdamC {
    float lr, b1, b2, r1, r2, eps;  // r1 = 1 / (1 - beta1^t), r2 = 1 / (1 - beta2^t)
};

// Adam over n parameters th (flat), gradient g in shared memory (same layout); the gradient is
// also stored to gout (the raw-gradient view).  With tgt != nullptr also the Polyak step of
// the matching target parameters, tgt <- tau theta_new + (1 - tau) tgt.  Four elements per
// thread per batch, loads before stores.
__device__ void adam_net(float* th, float* m, float* v, const float* g, int n, float* gout, const AdamC& A, float* tgt,
                         float tau)
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
                const float tn = tk[u] - A.lr * (mn * A.r1) / (sqrtf(vn * A.r2) + A.eps);
                gout[k] = gk[u];
                m[k] = mn;
                v[k] = vn;
                th[k] = tn;
                if (tgt) tgt[k] = fmaf(tau, tn, (1.0f - tau) * pk[u]);
            }
        }
    }
}

// Scratch per agent (floats): [0, B x 554): the actor's activation rows saved across the Q1
// pass (H1 at 0, H2 at 64 B: swizzled rows); then the raw gradients [Q1, Q2, actor] of the
// last update (read by the tests through TD3.grads(): they start at B x 554 floats).
__host__ __device__ inline int64_t td3_scratch_floats(int in_dim, int B)
{
    const int64_t f = (int64_t)B * 554 + 2 * net_size(kCI, 1) + net_size(in_dim, 4);
    return (f + 63) & ~(int64_t)63;  // every agent's scratch 256-byte aligned
}

__host__ __device__ inline int td3_wsm_floats(int in_dim)
{
    // the larger of: the actor net; both critic nets; a critic net + its gradient + the
    // output-layer gradient scratch (8 x 65 floats, wgrad_out)
    const int a = stage_floats(in_dim, 4), c = 2 * stage_floats(kCI, 1);
    const int g = stage_floats(kCI, 1) + net_size(kCI, 1) + 4 + 8 * (kH + 1);
    const int m = a > c ? a : c;
    return pad4(m > g ? m : g);
}

__host__ __device__ inline int64_t td3_smem_floats(int in_dim)
{
    return td3_wsm_floats(in_dim) + 2 * kB * kH + kB * kCI + kB * 4 + 32;
}

__global__ void __launch_bounds__(kT, 1) td3_update_kernel(TD3Dev A)
{
    extern __shared__ __align__(16) float sm[];
    const int ag = blockIdx.x, B = A.B, I = A.in_dim;
    const int s = threadIdx.x >> 1, hf = threadIdx.x & 1;  // per-sample helpers: sample, column half
    const bool act = s < B;
    const bool lead = act && hf == 0;
    const int sc = act ? s : B - 1;  // clamped sample index for inactive pairs' (discarded) loads
    const int64_t rb = (int64_t)ag * B + sc;
    const int na = net_size(I, 4), nc = net_size(kCI, 1);
    float* P = A.params + (int64_t)ag * A.block;
    const NetP actor = net_at(P, I, 4), actor_t = net_at(P + na, I, 4);
    const NetP Q0 = net_at(P + 2 * na, kCI, 1), Q1 = net_at(P + 2 * na + nc, kCI, 1);
    const NetP Qt0 = net_at(P + 2 * na + 2 * nc, kCI, 1), Qt1 = net_at(P + 2 * na + 3 * nc, kCI, 1);
    float* m_a = P + 2 * na + 4 * nc;
    float* v_a = m_a + na;
    float* scr = A.scratch + (int64_t)ag * A.scratch_floats;
    float* AH1 = scr;
    float* AH2 = scr + (int64_t)B * kH;
    float* gq0 = scr + (int64_t)B * 554;
    float* ga = gq0 + 2 * nc;
    const int S1c = wg_splits(kCI), S1a = wg_splits(I);

    float* Wsm = sm;
    float* Ab = Wsm + td3_wsm_floats(I);  // [kB][64] swizzled
    float* Bb = Ab + kB * kH;             // [kB][64] swizzled
    float* X32 = Bb + kB * kH;            // [kB][32] swizzled critic inputs
    float* D3 = X32 + kB * kCI;           // [kB][4] output-layer deltas
    float* red = D3 + kB * 4;             // [32]
    // gradients in shared memory (parameter layout): a critic's next to its staged net; the
    // actor's over its net once that is dead (W2/W3 parts first in X32, free at that point)
    const GradS Gc = grad_at(Wsm + stage_floats(kCI, 1), kCI, 1);
    const GradS Ga = grad_at(Wsm, I, 4);
    GradS Gt;  // (actor W2/b2/W3/b3 staging in X32: contiguous like the parameter layout)
    Gt.W2 = X32;
    Gt.b2 = Gt.W2 + kH * kH;
    Gt.W3 = Gt.b2 + kH;
    Gt.b3 = Gt.W3 + 4 * kH;
    Gt.W1 = Gt.b1 = nullptr;

#ifdef L2F_TD3_TIMING
    long long mark[16] = {};
#endif
    TD3_MARK(0);
    // ---- 1. target: a' = clip(pi'(o_a') + clip(sigma eps, -c, c), -1, 1); y = r + g (1-d) min Q'
    TD3_SUB(8);
    NetS W = fwd_input_layer(actor_t, Wsm, A.o_a2 + (int64_t)ag * B * I, I, B, Ab, Bb);
    own_rows_sync();
    TD3_SUB(9);
    fwd_gemm(Ab, kH, W.W2, kLd2, W.b2, Bb, B);
    own_rows_sync();
    TD3_SUB(10);
    {
        float at4[4];
        out_layer<4>(W, Bb, s, hf, at4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float nz = fminf(fmaxf(A.sigma_t * __ldg(A.eps + rb * 4 + k), -A.clip_t), A.clip_t);
            at4[k] = fminf(fmaxf(tanhf(at4[k]) + nz, -1.0f), 1.0f);
        }
        put_critic_row(X32, s, hf, A.o_c2 + rb * 28, at4);
    }
    __syncthreads();
    TD3_SUB(11);
    const NetS Wt0 = stage(Qt0, Wsm), Wt1 = stage(Qt1, Wsm + stage_floats(kCI, 1));
    __syncthreads();
    TD3_MARK(1);
    float qmin = 0.0f;
    for (int c = 0; c < 2; ++c) {
        const NetS& Wc = c == 0 ? Wt0 : Wt1;
        fwd_gemm(X32, kCI, Wc.W1, Wc.ld1, Wc.b1, Ab, B);
        own_rows_sync();
        fwd_gemm(Ab, kH, Wc.W2, kLd2, Wc.b2, Bb, B);
        own_rows_sync();
        float q[1];
        out_layer<1>(Wc, Bb, s, hf, q);
        qmin = c == 0 ? q[0] : fminf(qmin, q[0]);
    }
    const float y = __ldg(A.r + rb) + A.gamma * (1.0f - __ldg(A.done + rb)) * qmin;
    own_rows_sync();
    {  // the critic input rows (o_c, a), shared by both critics
        float a4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) a4[k] = __ldg(A.a + rb * 4 + k);
        put_critic_row(X32, s, hf, A.o_c + rb * 28, a4);
    }
    TD3_MARK(2);

    // ---- 2. critics: MSE to y, Adam (+ Polyak of the critic targets on delayed steps)
    const AdamC Ac{A.lr_critic, A.beta1, A.beta2, 1.0f / A.c1_critic, 1.0f / A.c2_critic, A.adam_eps};
    __syncthreads();
    W = stage(Q0, Wsm);
    for (int c = 0; c < 2; ++c) {  // (critic 1's net is prefetched during critic 0's Adam)
        const NetP& Qc = c == 0 ? Q0 : Q1;
        __syncthreads();
        fwd_gemm(X32, kCI, W.W1, W.ld1, W.b1, Ab, B);
        own_rows_sync();
        fwd_gemm(Ab, kH, W.W2, kLd2, W.b2, Bb, B);
        own_rows_sync();
        float q[1];
        out_layer<1>(W, Bb, s, hf, q);
        const float e = q[0] - y;
        const float d3[4] = {act ? 2.0f * e / (float)B : 0.0f, 0.f, 0.f, 0.f};
        if (lead) st4(D3 + 4 * s, make_float4(d3[0], 0.f, 0.f, 0.f));
        const float loss = block_sum(lead ? e * e / (float)B : 0.0f, red);  // (its barriers publish D3)
        if (threadIdx.x == 0) A.losses[ag * 3 + c] = loss;
        TD3_MARK(3 + 3 * c);
        net_backward(W, 1, D3, Ab, Bb, B, s, hf, d3, Gc, Gc, Gc.b3 + 4);  // (scratch after the gradient)
        // W1/b1: the ranges' partial tiles into the dead D2 buffer (Bb) and D3, one pass sums them
        wgrad<true>(Ab, X32, kCI, kCI, B, S1c, Gc.W1, Gc.b1, -1, true, Bb, D3);  // (ends with a barrier)
        TD3_MARK(4 + 3 * c);
        // prefetch the next phase's shared-memory operands under Adam's HBM traffic: critic 1's
        // net (beside the gradient this Adam reads), or the actor's input rows (free buffers;
        // nothing prefetched is updated by this Adam)
        if (c == 0)
            W = stage_issue(Q1, Wsm);
        else if (A.update_actor)
            input_rows_issue(A.o_a + (int64_t)ag * B * I, I, B, Ab, Bb);
        float* mc = m_a + 2 * na + 2 * c * nc;
        adam_net(Qc.W1, mc, mc + nc, Gc.W1, nc, gq0 + c * nc, Ac, A.update_actor ? (c == 0 ? Qt0 : Qt1).W1 : nullptr,
                 A.tau);
        if (c == 1 && A.update_actor) {
            __syncthreads();  // (every thread's Adam has read the gradient next to the net region)
            W = stage_issue(actor, Wsm);
        }
        cp_async_wait_all();
        TD3_MARK(5 + 3 * c);
    }
    if (!A.update_actor) {
        if (threadIdx.x == 0) A.losses[ag * 3 + 2] = 0.0f;
        return;
    }

    // ---- 3. actor: ascend Q1(o_c, pi(o_a)) through the updated Q1's action input, Adam + Polyak
    input_compute(W, I, B, Ab, Bb);  // (input rows staged during critic 1's Adam)
    const NetS Wa = W;
    // Q1 (the updated Q0 net) is staged under the actor's second layer where that leaves the
    // actor's W2/W3 intact for its backward: after the actor net, or over its (now dead) W1
    const int wsz = td3_wsm_floats(I), asz = stage_floats(I, 4), csz = stage_floats(kCI, 1);
    const int qoff = asz + csz <= wsz ? asz : (kH * ldw_of(I) + kH >= csz ? 0 : -1);
    NetS Wq;
    if (qoff >= 0) {
        __syncthreads();  // (every warp is done with the actor's W1)
        Wq = stage_issue(Q0, Wsm + qoff);
    }
    own_rows_sync();
    fwd_gemm(Ab, kH, W.W2, kLd2, W.b2, Bb, B);
    own_rows_sync();
    float ap[4];
    out_layer<4>(W, Bb, s, hf, ap);
#pragma unroll
    for (int k = 0; k < 4; ++k) ap[k] = tanhf(ap[k]);
    put_critic_row(X32, s, hf, A.o_c + rb * 28, ap);  // (o_c, pi(o_a))
    const int wr0 = 16 * (threadIdx.x >> 5), lane = threadIdx.x & 31;  // the warp's own rows
    for (int e = lane; e < 16 * kH / 4; e += 32) {  // save the actor's H1, H2 rows
        const int off = wr0 * kH + 4 * e;
        if (wr0 + (4 * e) / kH < B) {
            st4(AH1 + off, ld4(Ab + off));
            st4(AH2 + off, ld4(Bb + off));
        }
    }
    if (qoff < 0) {
        __syncthreads();
        Wq = stage_issue(Q0, Wsm);
    }
    cp_async_wait_all();
    __syncthreads();
    W = Wq;  // the updated Q1
    TD3_MARK(9);
    fwd_gemm(X32, kCI, W.W1, W.ld1, W.b1, Ab, B);
    own_rows_sync();
    fwd_gemm(Ab, kH, W.W2, kLd2, W.b2, Bb, B);
    own_rows_sync();
    float lossa;
    {
        float q[1];
        out_layer<1>(W, Bb, s, hf, q);
        lossa = lead ? -q[0] / (float)B : 0.0f;
        const float d3[1] = {-1.0f / (float)B};
        out_back<1>(W, Bb, s, hf, d3);
    }
    own_rows_sync();
    bwd_gemm(Bb, W.W2, Ab, B);
    own_rows_sync();
    float d3a[4];
    {  // dL/da = (W1^T d1)[28..31], d3a = dL/da (1 - a^2): my 32 rows of W1, pair-summed
        float da[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int c4 = 8 * hf + c;
            const float4 d = ld4(Ab + sw(s, c4, kH));
            const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float4 w = ld4(W.W1 + (4 * c4 + r) * W.ld1 + 28);
                da[0] = fmaf(w.x, dv[r], da[0]);
                da[1] = fmaf(w.y, dv[r], da[1]);
                da[2] = fmaf(w.z, dv[r], da[2]);
                da[3] = fmaf(w.w, dv[r], da[3]);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            da[k] += __shfl_xor_sync(0xffffffffu, da[k], 1);
            d3a[k] = act ? da[k] * (1.0f - ap[k] * ap[k]) : 0.0f;
        }
        if (lead) st4(D3 + 4 * s, make_float4(d3a[0], d3a[1], d3a[2], d3a[3]));
    }
    if (qoff < 0) {  // (the Q1 staging overwrote the actor's W2/W3)
        __syncthreads();
        W = stage(actor, Wsm);
    } else {
        own_rows_sync();
        W = Wa;
    }
    TD3_MARK(10);
    for (int e = lane; e < 16 * kH / 4; e += 32) {  // restore the actor's H1, H2 rows
        const int off = wr0 * kH + 4 * e;
        if (wr0 + (4 * e) / kH < B) {
            st4(Ab + off, ld4(AH1 + off));
            st4(Bb + off, ld4(AH2 + off));
        }
    }
    __syncthreads();
    net_backward(W, 4, D3, Ab, Bb, B, s, hf, d3a, Gt, Gt, Gt.b3 + 4);  // (W2/W3 gradients into X32)
    // the actor net is dead now: its W2/b2/W3/b3 gradient moves next to where W1's goes
    for (int e = threadIdx.x; e < (kH * kH + kH + 4 * kH + 4) / 4; e += blockDim.x) st4(Ga.W2 + 4 * e, ld4(Gt.W2 + 4 * e));
    for (int k0 = 0; k0 < I; k0 += kPW) {  // W1/b1 from staged column parts of o_a (into Bb + X32)
        const int w = min(kPW, pad4(I) - k0);
        __syncthreads();
        stage_cols(A.o_a + (int64_t)ag * B * I, B, I, k0, w, Bb);
        cp_async_wait_all();
        __syncthreads();
        wgrad<false>(Ab, Bb, kPLd, min(w, I - k0), B, S1a, Ga.W1 + k0, Ga.b1, I, k0 == 0);  // (ends with a barrier)
    }
    const float loss = block_sum(lossa, red);
    if (threadIdx.x == 0) A.losses[ag * 3 + 2] = loss;
    TD3_MARK(11);
    const AdamC Aa{A.lr_actor, A.beta1, A.beta2, 1.0f / A.c1_actor, 1.0f / A.c2_actor, A.adam_eps};
    adam_net(actor.W1, m_a, v_a, Ga.W1, na, ga, Aa, actor_t.W1, A.tau);  // ---- 4. with the actor target's Polyak step
    TD3_MARK(12);
#ifdef L2F_TD3_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        printf("L2F_TD3 target actor %lld target critics %lld critic0 fwd %lld bwd %lld adam %lld critic1 fwd %lld bwd "
               "%lld adam %lld actor fwd+Q1 %lld actor bwd %lld adam %lld total %lld\n",
               mark[1] - mark[0], mark[2] - mark[1], mark[3] - mark[2], mark[4] - mark[3], mark[5] - mark[4],
               mark[6] - mark[5], mark[7] - mark[6], mark[8] - mark[7], mark[10] - mark[8], mark[11] - mark[10],
               mark[12] - mark[11], mark[12] - mark[0]);
        printf("L2F_TD3 sub (actor phase): net + input staged %lld, input layer %lld | (target) L2 %lld | out+noise %lld"
               " | stage 2 critics %lld\n",
               g_td3_sub[0] - mark[9] + mark[9] - mark[8], g_td3_sub[1] - g_td3_sub[0], g_td3_sub[10] - g_td3_sub[9],
               g_td3_sub[11] - g_td3_sub[10], mark[1] - g_td3_sub[11]);
    }
#endif
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

int td3_max_in_dim() { return kMaxIn; }
int64_t td3_block_floats(int in_dim) { return 4 * (int64_t)net_size(in_dim, 4) + 8 * (int64_t)net_size(kCI, 1); }
int64_t td3_scratch_bytes(int in_dim, int B) { return 4 * td3_scratch_floats(in_dim, B); }

cudaError_t launch_td3_update(const TD3Dev& A, cudaStream_t s)
{
    if (A.B < 1 || A.B > kB || A.in_dim < 1 || A.in_dim > kMaxIn) return cudaErrorNotSupported;
    const size_t smem = (size_t)td3_smem_floats(A.in_dim) * sizeof(float);
    static std::atomic<size_t> attr[64] = {};
    const cudaError_t e = ensure_smem_attr(td3_update_kernel, smem, attr);
    if (e != cudaSuccess) return e;
    td3_update_kernel<<<A.n_agents, kT, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace l2f
