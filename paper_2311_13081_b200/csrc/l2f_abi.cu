// l2f_abi.cu -- extern "C" boundary of libl2f.so (include/l2f.h).
//
// Host-side responsibilities only: config validation, workspace carving, the curriculum
// stage table in FP64 -> fp32, launch-uniform parameter packing, and launches.
// Every step of the method itself runs in the kernels (l2f_kernels.cu, l2f_mlp.cu).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "../../include/l2f.h"
#include "l2f_internal.h"

using namespace l2f;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

l2f_status fail(l2f_status st, const std::string& msg)
{
    g_err = msg;
    return st;
}

l2f_status cuda_fail(cudaError_t e, const char* where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return L2F_ERR_CUDA;
}

// Every env entry point launches on the env's own device (the device of its workspace,
// recorded at l2f_create), whatever device is current in the calling thread; the caller's
// current device is restored on return (include/l2f.h conventions).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int32_t n_slots_for(int64_t n)
{
    const int64_t a = (n + kStepBlock - 1) / kStepBlock;
    const int64_t b = (n + kRolloutBlock - 1) / kRolloutBlock;
    const int64_t c = mlp_rollout_grid(n);
    int64_t m = a > b ? a : b;
    m = m > c ? m : c;
    return (int32_t)m;
}

constexpr size_t kPolicyMaxIn = 18 + 4 * L2F_MAX_HIST;
constexpr size_t kPolicyHalfs = 64 * kPolicyMaxIn + 64 + 64 * 64 + 64 + 4 * 64 + 4;

struct Layout {
    size_t state, dist, dr, hist, hist_t0, hist_fill, ep_step, ep_return, slots, stats_out, fin_part, st_act, st_obs,
        st_rew, st_flags, st_policy, total;
    int32_t n_slots;
};

Layout layout_for(const l2f_config& c)
{
    Layout L{};
    const size_t N = (size_t)c.num_envs;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    L.n_slots = n_slots_for(c.num_envs);
    L.state = take(4 * N * L2F_STATE_DIM);  // float4 groups + tail (DevBufs): exact bytes
    L.dist = take(4 * N * L2F_DIST_DIM);
    L.dr = take(4 * N * L2F_DR_DIM);
    L.hist = take(4 * N * 4 * (size_t)(c.action_history > 0 ? c.action_history : 1));
    L.hist_t0 = take(4 * N);
    L.hist_fill = take(4 * N * 4);
    L.ep_step = take(4 * N);
    L.ep_return = take(4 * N);
    L.slots = take(8 * (size_t)L.n_slots * L2F_STATS_LEN);
    L.stats_out = take(8 * L2F_STATS_LEN);
    L.fin_part = take(stats_finalize_scratch_bytes());  // partials + arrival ticket of the finalize reduction
    L.st_act = take(4 * N * 4);
    L.st_obs = take(4 * N * L2F_OBS_CORE);
    L.st_rew = take(4 * N);
    L.st_flags = take(N);
    L.st_policy = take(2 * kPolicyHalfs);
    L.total = o;
    return L;
}

l2f_status validate(const l2f_config* c)
{
    if (!c) return fail(L2F_ERR_INVALID_ARGUMENT, "config is NULL");
    if (c->abi_version != L2F_ABI_VERSION) return fail(L2F_ERR_INVALID_ARGUMENT, "abi_version mismatch");
    if (c->num_envs <= 0) return fail(L2F_ERR_INVALID_ARGUMENT, "num_envs must be > 0");
    if ((uint64_t)c->num_envs + c->env_id_offset > (1ull << 32))
        return fail(L2F_ERR_INVALID_ARGUMENT, "env_id_offset + num_envs must be <= 2^32 (Philox counter word)");
    if (c->action_history < 0 || c->action_history > L2F_MAX_HIST)
        return fail(L2F_ERR_INVALID_ARGUMENT, "action_history must be in [0, 32]");
    if (!(c->dt > 0)) return fail(L2F_ERR_INVALID_ARGUMENT, "dt must be > 0");
    if (c->max_episode_steps < 0) return fail(L2F_ERR_INVALID_ARGUMENT, "max_episode_steps must be >= 0");
    const l2f_params& p = c->params;
    if (!(p.rpm_max > p.rpm_min)) return fail(L2F_ERR_INVALID_ARGUMENT, "rpm_max must be > rpm_min");
    if (!(p.motor_tau > 0)) return fail(L2F_ERR_INVALID_ARGUMENT, "motor_tau must be > 0");
    if (!(p.mass > 0) || !(p.J[0] > 0) || !(p.J[1] > 0) || !(p.J[2] > 0))
        return fail(L2F_ERR_INVALID_ARGUMENT, "mass and inertia must be > 0");
    double lo = 1.0, hi = 1.0;
    if (c->flags & L2F_DOMAIN_RAND) {
        if (!(c->dr_lo > 0) || !(c->dr_hi >= c->dr_lo))
            return fail(L2F_ERR_INVALID_ARGUMENT, "DR range must satisfy 0 < dr_lo <= dr_hi");
        lo = c->dr_lo;
        hi = c->dr_hi;
    }
    // hover feasibility at the worst DR corner: 4 f(rpm_max) lo > m hi g
    const double w = p.rpm_max;
    const double f = p.thrust_c[0] + p.thrust_c[1] * w + p.thrust_c[2] * w * w;
    if (!(4.0 * f * lo > p.mass * hi * p.gravity))
        return fail(L2F_ERR_INVALID_ARGUMENT, "hover infeasible: 4 f(rpm_max) <= m g at the worst DR corner");
    if (c->init_rpm_lo > c->init_rpm_hi) return fail(L2F_ERR_INVALID_ARGUMENT, "init_rpm_lo > init_rpm_hi");
    if (c->curriculum.interval < 0) return fail(L2F_ERR_INVALID_ARGUMENT, "curriculum.interval must be >= 0");
    return L2F_OK;
}

// Curriculum stage k, FP64 on the host: w_k = clamp_toward(target, w_{k-1} * factor).
double toward(double w, double f, double target, double init)
{
    const double n = w * f;
    return init <= target ? std::fmin(n, target) : std::fmax(n, target);
}

StageW stage_weights(const l2f_config& c, int64_t k)
{
    const l2f_curriculum& C = c.curriculum;
    l2f_reward_weights w = C.init;
    double sg = C.sigma_init;
    // the schedule saturates after finitely many updates; iterate until fixed or k
    for (int64_t j = 0; j < k; ++j) {
        l2f_reward_weights n = w;
        n.C_rp = toward(w.C_rp, C.factor.C_rp, C.target.C_rp, C.init.C_rp);
        n.C_rq = toward(w.C_rq, C.factor.C_rq, C.target.C_rq, C.init.C_rq);
        n.C_rv = toward(w.C_rv, C.factor.C_rv, C.target.C_rv, C.init.C_rv);
        n.C_rw = toward(w.C_rw, C.factor.C_rw, C.target.C_rw, C.init.C_rw);
        n.C_ra = toward(w.C_ra, C.factor.C_ra, C.target.C_ra, C.init.C_ra);
        n.C_rs = toward(w.C_rs, C.factor.C_rs, C.target.C_rs, C.init.C_rs);
        const double ns = toward(sg, C.sigma_factor, C.sigma_target, C.sigma_init);
        const bool fixed = std::memcmp(&n, &w, sizeof(n)) == 0 && ns == sg;
        w = n;
        sg = ns;
        if (fixed) break;
    }
    StageW s;
    s.C_rp = (float)w.C_rp;
    s.C_rq = (float)w.C_rq;
    s.C_rv = (float)w.C_rv;
    s.C_rw = (float)w.C_rw;
    s.C_ra = (float)w.C_ra;
    for (int i = 0; i < 4; ++i) s.C_rab[i] = (float)w.C_rab[i];
    s.C_rs = (float)w.C_rs;
    s.sigma_a = (float)sg;
    return s;
}

}  // namespace

struct l2f_env {
    l2f_config cfg;
    int device;
    Layout L;
    uint8_t* ws;
    DevBufs B;
    DevParams base;
    uint64_t t;
    double steps;  // env-steps since the statistics were last reset (exact, host-side)
};

namespace {

DevParams make_base(const l2f_config& c)
{
    DevParams P;
    std::memset(&P, 0, sizeof(P));
    P.key0 = (uint32_t)c.seed;
    P.key1 = (uint32_t)(c.seed >> 32);
    for (int r = 0; r < 10; ++r) {  // Philox4x32-10 key schedule (Weyl constants)
        P.rk0[r] = P.key0 + (uint32_t)r * 0x9E3779B9u;
        P.rk1[r] = P.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    P.flags = c.flags;
    P.n_hist = c.action_history;
    P.max_ep = c.max_episode_steps;
    P.id_offset = (uint32_t)c.env_id_offset;
    P.n = c.num_envs;
    P.dt = (float)c.dt;
    P.half_dt = (float)(0.5 * c.dt);
    P.dt_6 = (float)(c.dt / 6.0);
    P.dt2_6 = (float)(c.dt * c.dt / 6.0);
    {  // RK4 of the rotor lag w' = (u - w)/T_m: stage factors and stability polynomial at z = dt/T_m
        const double z = c.dt / c.params.motor_tau;
        const double b2 = 1.0 - 0.5 * z, b3 = 1.0 - 0.5 * z * b2, b4 = 1.0 - z * b3;
        P.m_beta2 = (float)b2;
        P.m_beta3 = (float)b3;
        P.m_beta4 = (float)b4;
        P.m_R = (float)(1.0 - z / 6.0 * (1.0 + 2.0 * b2 + 2.0 * b3 + b4));
    }
    const l2f_params& p = c.params;
    P.mass = (float)p.mass;
    for (int j = 0; j < 3; ++j) {
        P.J[j] = (float)p.J[j];
        P.c[j] = (float)p.thrust_c[j];
    }
    P.ctau = (float)p.torque_c;
    P.inv_mass = (float)(1.0 / p.mass);
    for (int j = 0; j < 3; ++j) P.iJ[j] = (float)(1.0 / p.J[j]);
    P.dJ[0] = (float)p.J[2] - (float)p.J[1];  // same fp32 arithmetic as the DR path
    P.dJ[1] = (float)p.J[0] - (float)p.J[2];
    P.dJ[2] = (float)p.J[1] - (float)p.J[0];
    P.inv_tm = (float)(1.0 / p.motor_tau);
    P.rpm_min = (float)p.rpm_min;
    P.rpm_max = (float)p.rpm_max;
    P.gravity = (float)p.gravity;
    P.rpm_half_span = (float)(0.5 * (p.rpm_max - p.rpm_min));
    P.inv_rpm_span2 = (float)(2.0 / (p.rpm_max - p.rpm_min));
    for (int i = 0; i < 4; ++i) {
        P.rx[i] = (float)p.rotor_pos[i][0];
        P.ry[i] = (float)p.rotor_pos[i][1];
        P.spin[i] = (float)p.spin_dir[i];
        P.rxy[i] = make_float2(P.ry[i], -P.rx[i]);
    }
    P.init_pos = (float)c.init_pos;
    P.init_angle = (float)c.init_angle;
    P.init_vel = (float)c.init_vel;
    P.init_angvel = (float)c.init_angvel;
    P.init_rpm_lo = (float)c.init_rpm_lo;
    P.init_rpm_hi = (float)c.init_rpm_hi;
    P.dist_force = (float)c.dist_force;
    P.dist_torque = (float)c.dist_torque;
    P.dr_lo = (float)c.dr_lo;
    P.dr_hi = (float)c.dr_hi;
    {  // reset sampling table (reset_values): lo and the fp32-rounded span hi - lo per value
        auto rng = [](float lo, float hi, float4& L, float4& S, int k) {
            (&L.x)[k] = lo;
            (&S.x)[k] = hi - lo;  // fp32 subtraction, as a device-side hi - lo would round
        };
        const float pi2 = 6.28318530717958648f;
        for (int b = 0; b < 8; ++b) P.rs_lo[b] = P.rs_span[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < 3; ++k) rng(-P.init_pos, P.init_pos, P.rs_lo[0], P.rs_span[0], k);
        rng(-1.0f, 1.0f, P.rs_lo[0], P.rs_span[0], 3);                 // axis cos-polar
        P.rs_lo[1].x = 0.0f, P.rs_span[1].x = pi2;                      // axis azimuth
        P.rs_lo[1].y = 0.0f, P.rs_span[1].y = P.init_angle;             // rotation angle
        rng(-P.init_vel, P.init_vel, P.rs_lo[1], P.rs_span[1], 2);
        rng(-P.init_vel, P.init_vel, P.rs_lo[1], P.rs_span[1], 3);
        rng(-P.init_vel, P.init_vel, P.rs_lo[2], P.rs_span[2], 0);
        for (int k = 1; k < 4; ++k) rng(-P.init_angvel, P.init_angvel, P.rs_lo[2], P.rs_span[2], k);
        for (int k = 0; k < 4; ++k) rng(P.init_rpm_lo, P.init_rpm_hi, P.rs_lo[3], P.rs_span[3], k);
        for (int k = 0; k < 3; ++k) rng(-P.dist_force, P.dist_force, P.rs_lo[4], P.rs_span[4], k);
        rng(-P.dist_torque, P.dist_torque, P.rs_lo[4], P.rs_span[4], 3);
        for (int k = 0; k < 2; ++k) rng(-P.dist_torque, P.dist_torque, P.rs_lo[5], P.rs_span[5], k);
        for (int k = 0; k < 4; ++k) rng(P.dr_lo, P.dr_hi, P.rs_lo[6], P.rs_span[6], k);
        rng(P.dr_lo, P.dr_hi, P.rs_lo[7], P.rs_span[7], 0);
    }
    for (int j = 0; j < 4; ++j) P.obs_sigma[j] = (float)c.obs_sigma[j];
    P.term_pos = (float)c.term_pos;
    P.term_vel2 = (float)(c.term_vel * c.term_vel);
    P.term_angvel2 = (float)(c.term_angvel * c.term_angvel);
    return P;
}

// Launch parameters for steps [t0, t0 + T): the curriculum slice must fit kMaxStages.
bool params_for(const l2f_env* e, uint64_t t0, int64_t T, DevParams& P)
{
    P = e->base;
    P.t0 = (uint32_t)t0;
    P.hist_slot0 = e->cfg.action_history > 0 ? (int32_t)(t0 % (uint64_t)e->cfg.action_history) : 0;
    const int64_t I = e->cfg.curriculum.interval;
    int64_t k0 = 0, k1 = 0;
    if (I > 0) {
        k0 = (int64_t)(t0 / (uint64_t)I);
        k1 = (int64_t)((t0 + (uint64_t)(T > 0 ? T - 1 : 0)) / (uint64_t)I);
    }
    if (k1 - k0 + 1 > kMaxStages) return false;
    P.n_stages = (int32_t)(k1 - k0 + 1);
    for (int64_t k = k0; k <= k1; ++k) {
        P.stage[k - k0] = stage_weights(e->cfg, k);
        P.stage_end[k - k0] = (uint32_t)((k + 1) * (I > 0 ? I : 0));  // stage k covers [k I, (k+1) I)
    }
    return true;
}

StepOutDev to_dev(const l2f_step_out* o)
{
    StepOutDev d{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    if (o) {
        d.obs_core = o->obs_core;
        d.obs_dense = o->obs_dense;
        d.reward = o->reward;
        d.flags = o->flags;
        d.final_state = o->final_state;
        d.obs_critic = o->obs_critic;
    }
    return d;
}

l2f_status launched(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) return cuda_fail(e, what);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return L2F_OK;
}

}  // namespace

extern "C" {

int32_t l2f_abi_version(void) { return L2F_ABI_VERSION; }

const char* l2f_last_error(void) { return g_err.c_str(); }

uint64_t l2f_launch_count(void) { return g_launches.load(); }

l2f_status l2f_workspace_size(const l2f_config* cfg, size_t* bytes)
{
    l2f_status st = validate(cfg);
    if (st != L2F_OK) return st;
    if (!bytes) return fail(L2F_ERR_INVALID_ARGUMENT, "bytes is NULL");
    *bytes = layout_for(*cfg).total;
    return L2F_OK;
}

l2f_status l2f_create(const l2f_config* cfg, void* d_workspace, size_t bytes, l2f_env** out)
{
    l2f_status st = validate(cfg);
    if (st != L2F_OK) return st;
    if (!out || !d_workspace) return fail(L2F_ERR_INVALID_ARGUMENT, "out/workspace is NULL");
    if (((uintptr_t)d_workspace) & 255) return fail(L2F_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    Layout L = layout_for(*cfg);
    if (bytes < L.total) return fail(L2F_ERR_WORKSPACE_TOO_SMALL, "workspace smaller than l2f_workspace_size()");
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, d_workspace);
    if (e != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return fail(L2F_ERR_INVALID_ARGUMENT, "workspace is not CUDA device memory");
    }
    l2f_env* env = new (std::nothrow) l2f_env;
    if (!env) return fail(L2F_ERR_BAD_STATE, "out of host memory");
    env->cfg = *cfg;
    env->device = attr.device;
    env->L = L;
    env->ws = (uint8_t*)d_workspace;
    env->B.state = (float4*)(env->ws + L.state);
    env->B.dist = (float4*)(env->ws + L.dist);
    env->B.dr = (float4*)(env->ws + L.dr);
    env->B.hist = (float4*)(env->ws + L.hist);
    env->B.hist_t0 = (int32_t*)(env->ws + L.hist_t0);
    env->B.hist_fill = (float4*)(env->ws + L.hist_fill);
    env->B.ep_step = (int32_t*)(env->ws + L.ep_step);
    env->B.ep_return = (float*)(env->ws + L.ep_return);
    env->B.slots = (double*)(env->ws + L.slots);
    env->B.n_slots = L.n_slots;
    env->base = make_base(*cfg);
    env->t = 0;
    env->steps = 0.0;
    *out = env;
    return L2F_OK;
}

l2f_status l2f_destroy(l2f_env* env)
{
    delete env;
    return L2F_OK;
}

l2f_status l2f_reset(l2f_env* env, const uint8_t* d_mask, const l2f_step_out* out, void* stream)
{
    if (!env) return fail(L2F_ERR_INVALID_ARGUMENT, "env is NULL");
    const DeviceGuard guard(env->device);
    cudaStream_t s = (cudaStream_t)stream;
    DevParams P;
    params_for(env, env->t, 1, P);
    if (!d_mask) {
        // full reset: statistics and the (lazily overwritten) history ring start from zero, so
        // the whole workspace state is a deterministic function of (config, t, actions)
        cudaError_t e = cudaMemsetAsync(env->B.slots, 0, sizeof(double) * L2F_STATS_LEN * env->L.n_slots, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(env->ws + env->L.fin_part, 0, stats_finalize_scratch_bytes(), s);
        if (e == cudaSuccess && env->cfg.action_history > 0)
            e = cudaMemsetAsync(env->B.hist, 0, sizeof(float) * 4 * (size_t)env->cfg.action_history * env->cfg.num_envs, s);
        if (e != cudaSuccess) return cuda_fail(e, "l2f_reset memset");
        env->steps = 0.0;
    }
    return launched(launch_reset(P, env->B, d_mask, to_dev(out), s), "l2f_reset");
}

l2f_status l2f_step(l2f_env* env, const float* d_actions, const l2f_step_out* out, void* stream)
{
    if (!env || !d_actions) return fail(L2F_ERR_INVALID_ARGUMENT, "env/actions is NULL");
    const DeviceGuard guard(env->device);
    DevParams P;
    params_for(env, env->t, 1, P);
    l2f_status st = launched(launch_step(P, env->B, d_actions, to_dev(out), (cudaStream_t)stream), "l2f_step");
    if (st == L2F_OK) {
        env->t += 1;
        env->steps += (double)env->cfg.num_envs;
    }
    return st;
}

l2f_status l2f_rollout(l2f_env* env, const l2f_policy* policy, const float* d_actions, int32_t T, float* d_trace,
                       const int64_t* d_trace_ids, int32_t K, void* stream)
{
    if (!env) return fail(L2F_ERR_INVALID_ARGUMENT, "env is NULL");
    const DeviceGuard guard(env->device);
    if (T < 1) return fail(L2F_ERR_INVALID_ARGUMENT, "T must be >= 1");
    if (d_trace && (!d_trace_ids || K < 1 || K > 4096))
        return fail(L2F_ERR_INVALID_ARGUMENT, "trace needs trace ids and 1 <= K <= 4096");
    if (policy && d_actions) return fail(L2F_ERR_INVALID_ARGUMENT, "policy and actions are exclusive");
    if (policy) {
        const int32_t nh = env->cfg.action_history;
        if (policy->in_dim != 18 + 4 * nh || policy->hidden != 64)
            return fail(L2F_ERR_INVALID_ARGUMENT, "policy must be (18 + 4 N_H) -> 64 -> 64 -> 4");
        if (nh % 4 != 0) return fail(L2F_ERR_NOT_SUPPORTED, "MLP rollout needs N_H % 4 == 0");
        if (!policy->W1 || !policy->b1 || !policy->W2 || !policy->b2 || !policy->W3 || !policy->b3)
            return fail(L2F_ERR_INVALID_ARGUMENT, "policy pointer is NULL");
    }
    cudaStream_t s = (cudaStream_t)stream;
    // split so every launch sees at most kMaxStages curriculum stages
    int32_t done = 0;
    while (done < T) {
        // (the rollouts' packed per-thread statistics hold <= 65535 steps per launch)
        int32_t chunk = T - done < 65535 ? T - done : 65535;
        DevParams P;
        while (!params_for(env, env->t, chunk, P)) chunk = chunk / 2 > 0 ? chunk / 2 : 1;
        float* tr = d_trace ? d_trace + (size_t)done * K * L2F_TRACE_FIELDS : nullptr;
        cudaError_t e;
        if (policy) {
            PolicyDev W{policy->W1, policy->b1, policy->W2, policy->b2, policy->W3, policy->b3, policy->in_dim,
                        policy->hidden};
            e = launch_rollout_mlp(P, env->B, W, chunk, tr, d_trace_ids, K, s);
        } else {
            const float* a = d_actions ? d_actions + (size_t)done * 4 * env->cfg.num_envs : nullptr;
            e = launch_rollout_open(P, env->B, a, chunk, tr, d_trace_ids, K, s);
        }
        if (e == cudaErrorNotSupported) return fail(L2F_ERR_NOT_SUPPORTED, "rollout configuration not supported");
        l2f_status st = launched(e, "l2f_rollout");
        if (st != L2F_OK) return st;
        env->t += (uint64_t)chunk;
        env->steps += (double)chunk * (double)env->cfg.num_envs;
        done += chunk;
    }
    return L2F_OK;
}

l2f_status l2f_track(l2f_env* env, const l2f_policy* policy, const l2f_tracking* spec, void* stream)
{
    if (!env || !policy || !spec) return fail(L2F_ERR_INVALID_ARGUMENT, "env/policy/spec is NULL");
    const DeviceGuard guard(env->device);
    if (!spec->cycle_time || !spec->rmse || !spec->rmse_xy || !spec->steps_ok)
        return fail(L2F_ERR_INVALID_ARGUMENT, "tracking buffers must not be NULL");
    if (spec->n_steps < 1 || !(spec->clip_pos > 0) || !(spec->clip_vel > 0))
        return fail(L2F_ERR_INVALID_ARGUMENT, "tracking needs n_steps >= 1 and positive clip bounds");
    const int32_t nh = env->cfg.action_history;
    if (policy->in_dim != 18 + 4 * nh || policy->hidden != 64)
        return fail(L2F_ERR_INVALID_ARGUMENT, "policy must be (18 + 4 N_H) -> 64 -> 64 -> 4");
    if (nh % 4 != 0) return fail(L2F_ERR_NOT_SUPPORTED, "tracking needs N_H % 4 == 0");
    if (!policy->W1 || !policy->b1 || !policy->W2 || !policy->b2 || !policy->W3 || !policy->b3)
        return fail(L2F_ERR_INVALID_ARGUMENT, "policy pointer is NULL");
    if (env->t + (uint64_t)spec->n_steps >= (1ull << 31)) return fail(L2F_ERR_INVALID_ARGUMENT, "t overflow");
    DevParams P;
    params_for(env, env->t, 1, P);  // stage weights are irrelevant here (no reward output)
    const uint32_t keep = F_OBS_NOISE | F_NO_ROTOR_DELAY;  // deterministic actor, no resets / DR / disturbance
    const bool terminate = (P.flags & F_TERMINATION) != 0;
    P.flags &= keep;
    // hover rotor speed of the nominal parameters: 4 (c0 + c1 w + c2 w^2) = m g
    const l2f_params& pp = env->cfg.params;
    const double c0 = pp.thrust_c[0] - pp.mass * pp.gravity / 4.0, c1 = pp.thrust_c[1], c2 = pp.thrust_c[2];
    const double wh = c2 != 0.0 ? (-c1 + std::sqrt(c1 * c1 - 4.0 * c2 * c0)) / (2.0 * c2) : -c0 / c1;
    TrackDev S;
    S.cycle_time = spec->cycle_time;
    S.ax = (float)spec->amp_x;
    S.ay = (float)spec->amp_y;
    S.z = (float)spec->altitude;
    S.clip_pos = (float)spec->clip_pos;
    S.clip_vel = (float)spec->clip_vel;
    S.hover_rpm = (float)wh;
    S.hover_a = (float)(2.0 * (wh - pp.rpm_min) / (pp.rpm_max - pp.rpm_min) - 1.0);
    S.n_steps = spec->n_steps;
    S.terminate = terminate ? 1 : 0;
    S.rmse = spec->rmse;
    S.rmse_xy = spec->rmse_xy;
    S.steps_ok = spec->steps_ok;
    PolicyDev W{policy->W1, policy->b1, policy->W2, policy->b2, policy->W3, policy->b3, policy->in_dim,
                policy->hidden};
    const cudaError_t e = launch_track_mlp(P, env->B, W, S, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) return fail(L2F_ERR_NOT_SUPPORTED, "tracking configuration not supported");
    const l2f_status st = launched(e, "l2f_track");
    if (st == L2F_OK) env->t += (uint64_t)spec->n_steps;
    return st;
}

l2f_status l2f_td3_sizes(int32_t in_dim, int32_t batch, int64_t* block_floats, int64_t* scratch_bytes_per_agent)
{
    if (in_dim < 1 || in_dim > td3_max_in_dim() || batch < 1 || batch > 256)
        return fail(L2F_ERR_INVALID_ARGUMENT, "TD3 needs 1 <= in_dim <= 156 and 1 <= batch <= 256");
    if (block_floats) *block_floats = td3_block_floats(in_dim);
    if (scratch_bytes_per_agent) *scratch_bytes_per_agent = td3_scratch_bytes(in_dim, batch);
    return L2F_OK;
}

l2f_status l2f_td3_update(float* d_params, int32_t n_agents, int32_t in_dim, int32_t batch, const l2f_td3_batch* b,
                          const l2f_td3_hyper* h, int64_t t_critic, int64_t t_actor, int32_t update_actor,
                          float* d_losses, void* d_scratch, void* stream)
{
    int64_t blk = 0, sb = 0;
    l2f_status st = l2f_td3_sizes(in_dim, batch, &blk, &sb);
    if (st != L2F_OK) return st;
    if (!d_params || !b || !h || !d_losses || !d_scratch || n_agents < 1)
        return fail(L2F_ERR_INVALID_ARGUMENT, "bad TD3 arguments");
    if (!b->o_a || !b->o_c || !b->a || !b->r || !b->o_a2 || !b->o_c2 || !b->done || !b->eps)
        return fail(L2F_ERR_INVALID_ARGUMENT, "TD3 batch pointer is NULL");
    if (t_critic < 1 || (update_actor && t_actor < 1)) return fail(L2F_ERR_INVALID_ARGUMENT, "Adam steps start at 1");
    if (!(h->gamma >= 0 && h->gamma <= 1) || !(h->tau >= 0 && h->tau <= 1) || !(h->beta1 >= 0 && h->beta1 < 1) ||
        !(h->beta2 >= 0 && h->beta2 < 1) || !(h->eps > 0))
        return fail(L2F_ERR_INVALID_ARGUMENT, "bad TD3 hyper-parameters");
    TD3Dev A;
    A.params = d_params;
    A.scratch = (float*)d_scratch;
    A.losses = d_losses;
    A.o_a = b->o_a;
    A.o_c = b->o_c;
    A.a = b->a;
    A.r = b->r;
    A.o_a2 = b->o_a2;
    A.o_c2 = b->o_c2;
    A.done = b->done;
    A.eps = b->eps;
    A.block = blk;
    A.scratch_floats = sb / 4;
    A.n_agents = n_agents;
    A.B = batch;
    A.in_dim = in_dim;
    A.update_actor = update_actor ? 1 : 0;
    A.gamma = (float)h->gamma;
    A.tau = (float)h->tau;
    A.sigma_t = (float)h->sigma_t;
    A.clip_t = (float)h->clip_t;
    A.lr_actor = (float)h->lr_actor;
    A.lr_critic = (float)h->lr_critic;
    A.beta1 = (float)h->beta1;
    A.beta2 = (float)h->beta2;
    A.adam_eps = (float)h->eps;
    A.c1_critic = (float)(1.0 - std::pow(h->beta1, (double)t_critic));
    A.c2_critic = (float)(1.0 - std::pow(h->beta2, (double)t_critic));
    A.c1_actor = (float)(1.0 - std::pow(h->beta1, (double)(t_actor > 0 ? t_actor : 1)));
    A.c2_actor = (float)(1.0 - std::pow(h->beta2, (double)(t_actor > 0 ? t_actor : 1)));
    const cudaError_t e = launch_td3_update(A, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) return fail(L2F_ERR_NOT_SUPPORTED, "TD3 configuration not supported");
    return launched(e, "l2f_td3_update");
}

l2f_status l2f_td3_export_actor(const float* d_params, int32_t agent, int32_t in_dim, uint16_t* d_out,
                                l2f_policy* out, void* stream)
{
    if (!d_params || !d_out || !out || agent < 0 || in_dim < 1 || in_dim > 256)
        return fail(L2F_ERR_INVALID_ARGUMENT, "bad td3_export_actor arguments");
    const cudaError_t e = launch_td3_export_actor(d_params, td3_block_floats(in_dim), agent, in_dim, d_out,
                                                  (cudaStream_t)stream);
    const int64_t H = 64;
    out->W1 = d_out;
    out->b1 = out->W1 + H * in_dim;
    out->W2 = out->b1 + H;
    out->b2 = out->W2 + H * H;
    out->W3 = out->b2 + H;
    out->b3 = out->W3 + 4 * H;
    out->in_dim = in_dim;
    out->hidden = (int32_t)H;
    return launched(e, "l2f_td3_export_actor");
}

l2f_status l2f_episode_stats(l2f_env* env, double* d_out, int32_t reset_accumulators, void* stream)
{
    if (!env || !d_out) return fail(L2F_ERR_INVALID_ARGUMENT, "env/out is NULL");
    const DeviceGuard guard(env->device);
    l2f_status st = launched(launch_stats_finalize(env->B.slots, env->L.n_slots, env->ws + env->L.fin_part, d_out,
                                                   reset_accumulators,
                                                   env->steps, (cudaStream_t)stream),
                             "l2f_episode_stats");
    if (st == L2F_OK && reset_accumulators) env->steps = 0.0;
    return st;
}

l2f_status l2f_step_host(l2f_env* env, const float* h_actions, float* h_obs_core, float* h_reward, uint8_t* h_flags,
                         void* stream)
{
    if (!env || !h_actions) return fail(L2F_ERR_INVALID_ARGUMENT, "env/actions is NULL");
    const DeviceGuard guard(env->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t N = (size_t)env->cfg.num_envs;
    float* d_act = (float*)(env->ws + env->L.st_act);
    l2f_step_out o{};
    o.obs_core = h_obs_core ? (float*)(env->ws + env->L.st_obs) : nullptr;
    o.reward = h_reward ? (float*)(env->ws + env->L.st_rew) : nullptr;
    o.flags = h_flags ? (uint8_t*)(env->ws + env->L.st_flags) : nullptr;
    cudaError_t e = cudaMemcpyAsync(d_act, h_actions, 4 * N * sizeof(float), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "l2f_step_host H2D");
    l2f_status st = l2f_step(env, d_act, &o, stream);
    if (st != L2F_OK) return st;
    if (h_obs_core &&
        (e = cudaMemcpyAsync(h_obs_core, o.obs_core, L2F_OBS_CORE * N * sizeof(float), cudaMemcpyDeviceToHost, s)))
        return cuda_fail(e, "l2f_step_host D2H obs");
    if (h_reward && (e = cudaMemcpyAsync(h_reward, o.reward, N * sizeof(float), cudaMemcpyDeviceToHost, s)))
        return cuda_fail(e, "l2f_step_host D2H reward");
    if (h_flags && (e = cudaMemcpyAsync(h_flags, o.flags, N, cudaMemcpyDeviceToHost, s)))
        return cuda_fail(e, "l2f_step_host D2H flags");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "l2f_step_host sync");
    return L2F_OK;
}

l2f_status l2f_rollout_host(l2f_env* env, const l2f_policy* h_policy, int32_t T, double* h_stats,
                            int32_t reset_accumulators, void* stream)
{
    if (!env || !h_policy) return fail(L2F_ERR_INVALID_ARGUMENT, "env/policy is NULL");
    const DeviceGuard guard(env->device);
    const int32_t I = h_policy->in_dim, H = h_policy->hidden;
    if (I != 18 + 4 * env->cfg.action_history || H != 64)
        return fail(L2F_ERR_INVALID_ARGUMENT, "policy must be (18 + 4 N_H) -> 64 -> 64 -> 4");
    cudaStream_t s = (cudaStream_t)stream;
    uint16_t* base = (uint16_t*)(env->ws + env->L.st_policy);
    const size_t n1 = (size_t)H * I, n2 = (size_t)H * H, n3 = 4 * (size_t)H;
    uint16_t* W1 = base;
    uint16_t* b1 = W1 + n1;
    uint16_t* W2 = b1 + H;
    uint16_t* b2 = W2 + n2;
    uint16_t* W3 = b2 + H;
    uint16_t* b3 = W3 + n3;
    const struct {
        uint16_t* d;
        const uint16_t* h;
        size_t n;
    } cp[6] = {{W1, h_policy->W1, n1}, {b1, h_policy->b1, (size_t)H}, {W2, h_policy->W2, n2},
               {b2, h_policy->b2, (size_t)H}, {W3, h_policy->W3, n3}, {b3, h_policy->b3, 4}};
    for (auto& c : cp) {
        if (!c.h) return fail(L2F_ERR_INVALID_ARGUMENT, "policy pointer is NULL");
        cudaError_t e = cudaMemcpyAsync(c.d, c.h, c.n * 2, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "l2f_rollout_host H2D policy");
    }
    l2f_policy dp{W1, b1, W2, b2, W3, b3, I, H};
    l2f_status st = l2f_rollout(env, &dp, nullptr, T, nullptr, nullptr, 0, stream);
    if (st != L2F_OK) return st;
    double* d_stats = (double*)(env->ws + env->L.stats_out);
    st = l2f_episode_stats(env, d_stats, reset_accumulators, stream);
    if (st != L2F_OK) return st;
    cudaError_t e;
    if (h_stats &&
        (e = cudaMemcpyAsync(h_stats, d_stats, L2F_STATS_LEN * sizeof(double), cudaMemcpyDeviceToHost, s)))
        return cuda_fail(e, "l2f_rollout_host D2H stats");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "l2f_rollout_host sync");
    return L2F_OK;
}

l2f_status l2f_get_state(l2f_env* env, l2f_state_view* out)
{
    if (!env || !out) return fail(L2F_ERR_INVALID_ARGUMENT, "env/out is NULL");
    out->state = (float*)env->B.state;
    out->dist = (float*)env->B.dist;
    out->dr = (float*)env->B.dr;
    out->hist = (float*)env->B.hist;
    out->hist_t0 = env->B.hist_t0;
    out->hist_fill = (float*)env->B.hist_fill;
    out->ep_step = env->B.ep_step;
    out->ep_return = env->B.ep_return;
    out->t = env->t;
    out->num_envs = env->cfg.num_envs;
    out->action_history = env->cfg.action_history;
    return L2F_OK;
}

l2f_status l2f_set_t(l2f_env* env, uint64_t t)
{
    if (!env) return fail(L2F_ERR_INVALID_ARGUMENT, "env is NULL");
    if (t >= (1ull << 31)) return fail(L2F_ERR_INVALID_ARGUMENT, "t must be < 2^31");
    env->t = t;
    return L2F_OK;
}

l2f_status l2f_set_state(l2f_env* env, const l2f_state_view* in, void* stream)
{
    if (!env || !in) return fail(L2F_ERR_INVALID_ARGUMENT, "env/in is NULL");
    const DeviceGuard guard(env->device);
    const int64_t N = env->cfg.num_envs;
    const int32_t NH = env->cfg.action_history;
    if (in->num_envs != N || in->action_history != NH)
        return fail(L2F_ERR_INVALID_ARGUMENT, "set_state: num_envs/action_history differ from the env's");
    if (in->t >= (1ull << 31)) return fail(L2F_ERR_INVALID_ARGUMENT, "t must be < 2^31");
    const cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)N;
    struct Part {
        void* dst;
        const void* src;
        size_t bytes;
    } parts[] = {
        {env->B.state, in->state, 4 * n * L2F_STATE_DIM},
        {env->B.dist, in->dist, 4 * n * L2F_DIST_DIM},
        {env->B.dr, in->dr, 4 * n * L2F_DR_DIM},
        {env->B.hist, in->hist, 4 * n * 4 * (size_t)(NH > 0 ? NH : 1)},
        {env->B.hist_t0, in->hist_t0, 4 * n},
        {env->B.hist_fill, in->hist_fill, 4 * n * 4},
        {env->B.ep_step, in->ep_step, 4 * n},
        {env->B.ep_return, in->ep_return, 4 * n},
    };
    for (const Part& p : parts) {
        if (!p.src || p.src == p.dst) continue;
        const cudaError_t e = cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return fail(L2F_ERR_CUDA, cudaGetErrorString(e));
    }
    env->t = in->t;
    return L2F_OK;
}

l2f_status l2f_policy_forward(const l2f_policy* policy, const float* d_obs, float* d_act, int64_t n, void* stream)
{
    if (!policy || !d_obs || !d_act || n <= 0) return fail(L2F_ERR_INVALID_ARGUMENT, "bad policy_forward arguments");
    if (policy->hidden != 64 || policy->in_dim < 18 || ((policy->in_dim - 18) % 16) != 0 ||
        policy->in_dim > 18 + 4 * L2F_MAX_HIST)
        return fail(L2F_ERR_NOT_SUPPORTED, "policy_forward needs hidden 64 and in_dim = 18 + 16 j <= 146");
    PolicyDev W{policy->W1, policy->b1, policy->W2, policy->b2, policy->W3, policy->b3, policy->in_dim,
                policy->hidden};
    cudaError_t e = launch_policy_forward(W, d_obs, d_act, n, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) return fail(L2F_ERR_NOT_SUPPORTED, "policy_forward not supported");
    return launched(e, "l2f_policy_forward");
}

l2f_status l2f_recompute_rewards(const l2f_env* env, uint64_t t, const float* d_next_state, const float* d_actions,
                                 int64_t m, float* d_rewards, void* stream)
{
    if (!env || !d_next_state || !d_actions || !d_rewards || m <= 0)
        return fail(L2F_ERR_INVALID_ARGUMENT, "bad recompute_rewards arguments");
    const DeviceGuard guard(env->device);
    const int64_t I = env->cfg.curriculum.interval;
    const int64_t k = I > 0 ? (int64_t)(t / (uint64_t)I) : 0;
    const StageW W = stage_weights(env->cfg, k);
    return launched(launch_recompute_rewards(W, d_next_state, d_actions, m, d_rewards, (cudaStream_t)stream),
                    "l2f_recompute_rewards");
}

l2f_status l2f_selftest_philox(int64_t n, uint64_t seed, uint32_t t, uint32_t* d_ours, uint32_t* d_curand,
                               void* stream)
{
    if (n <= 0 || !d_ours || !d_curand) return fail(L2F_ERR_INVALID_ARGUMENT, "bad selftest arguments");
    return launched(launch_philox_selftest(n, seed, t, d_ours, d_curand, (cudaStream_t)stream), "l2f_selftest_philox");
}

}  // extern "C"
