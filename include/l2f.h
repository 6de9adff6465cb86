/*
 * l2f.h -- C ABI of the B200-native batched quadrotor environment of arXiv 2311.13081
 * ("Learning to Fly in Seconds").  libl2f.so, sm_100a.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n.  "Qn" = a reading of the paper listed
 * in DESIGN.md section 3 (where the paper is silent).
 *
 * The library computes, for N independent environments, the MDP of P:131-152:
 *   state  s = {p, q, v, omega, omega_m} (17-D), per-episode disturbance
 *          {f_r, tau_r}, optional per-env domain-randomised parameters (Q19);
 *   action a in [-1,1]^4 = normalised RPM setpoints;
 *   step   first-order motor lag + polynomial RPM->thrust/torque
 *          + rigid-body dynamics integrated with RK4 at dt (Q1);
 *   obs    o_a = {p, R(q), v, omega, H} + noise, H = action history;
 *   reward r(s,a,s') with curriculum-scheduled weights;
 *   done   termination (Q14) / truncation (Q15), same-step auto-reset (Q16).
 * and a fused rollout that evaluates the actor MLP per env between steps.
 *
 * Conventions for every entry point:
 *  - All functions are extern "C", never throw, and return an l2f_status.  On a non-OK
 *    status l2f_last_error() returns a thread-local message.
 *  - Device pointers ("d_") are caller-owned CUDA device memory on the env's device; host
 *    pointers ("h_") are caller-owned host memory.  An env's device is the device of its
 *    workspace; every call on an env launches there whatever device is current in the
 *    calling thread (the current device is restored on return), so `stream` must be a
 *    stream of that device (or NULL, its legacy default stream).  The library never allocates device
 *    memory: the caller provides a workspace of l2f_workspace_size() bytes at create time.
 *  - Every call is asynchronous on the caller's stream (a cudaStream_t passed as void*;
 *    NULL = the legacy default stream) unless its comment says it synchronises.  The
 *    returned status covers argument validation and launch errors; asynchronous device
 *    faults surface at the caller's next synchronisation.
 *  - Layouts are structure-of-arrays: "[C][N]" means component-major, env index fastest
 *    (element (c, i) at c*N + i), fp32 unless stated.
 *  - Numerical divergence (non-finite state) is per env, never a global error: the env
 *    is flagged L2F_DONE_DIVERGED | L2F_DONE_TERMINATED.
 */
#ifndef L2F_H
#define L2F_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define L2F_API __attribute__((visibility("default")))
#else
#define L2F_API
#endif

#define L2F_ABI_VERSION 2
#define L2F_STATE_DIM 17     /* p(3) q(4: w,x,y,z) v(3) omega(3) omega_m(4) */
#define L2F_OBS_CORE 18      /* p(3) R(9, row-major) v(3) omega(3) */
#define L2F_MAX_HIST 32      /* N_H upper bound                                  */
#define L2F_DIST_DIM 6       /* f_r (world, N), tau_r (body, N m) */
#define L2F_DR_DIM 5         /* mass, Jxx, Jyy, Jzz, thrust-curve scale factors (Q19)  */
#define L2F_STATS_LEN 8
#define L2F_TRACE_FIELDS 32

typedef struct l2f_env l2f_env; /* opaque */

typedef enum {
    L2F_OK = 0,
    L2F_ERR_INVALID_ARGUMENT = 1,
    L2F_ERR_CUDA = 2,
    L2F_ERR_WORKSPACE_TOO_SMALL = 3,
    L2F_ERR_NOT_SUPPORTED = 4,
    L2F_ERR_BAD_STATE = 5
} l2f_status;

/* Feature flags (l2f_config.flags). */
enum {
    L2F_OBS_NOISE = 1u << 0,      /* Gaussian observation noise on p, R, v, omega   */
    L2F_ACTION_NOISE = 1u << 1,   /* Gaussian exploration noise on actions (Q7)      */
    L2F_TERMINATION = 1u << 2,    /* box / speed termination (Q14)                   */
    L2F_AUTO_RESET = 1u << 3,     /* same-step reset of ended envs (Q16)                    */
    L2F_DISTURBANCE = 1u << 4,    /* per-episode random force/torque                */
    L2F_DOMAIN_RAND = 1u << 5,    /* per-episode mass/inertia/thrust factors (Q19)          */
    L2F_NO_ROTOR_DELAY = 1u << 6  /* ablation (Table II "Rotor Delay"): the rotor
                                     speeds are set to the setpoint at the start of each step
                                      instead of following the first-order lag       */
};

/* Per-env step flags (l2f_step_out.flags, trace field 26). */
enum { L2F_DONE_TERMINATED = 1, L2F_DONE_TRUNCATED = 2, L2F_DONE_DIVERGED = 4, L2F_DONE_RESET = 8 };

/* Episode statistics (l2f_episode_stats output, FP64). */
enum {
    L2F_ST_EPISODES = 0,  /* episodes that ended (terminated or truncated)   */
    L2F_ST_TERMINATED,
    L2F_ST_TRUNCATED,
    L2F_ST_DIVERGED,
    L2F_ST_SUM_LEN,       /* sum of episode lengths (steps)                  */
    L2F_ST_SUM_RET,       /* sum of episode returns                          */
    L2F_ST_SUM_RET_SQ,    /* sum of squared episode returns                  */
    L2F_ST_ENV_STEPS      /* env-steps executed                              */
};

/* Quadrotor parameters. m = 0.027 kg and T_m = 0.15 s are the paper's. */
typedef struct {
    double mass;            /* kg */
    double J[3];            /* diagonal inertia, kg m^2 */
    double rotor_pos[4][3]; /* body frame, m */
    double spin_dir[4];     /* +1 / -1 */
    double thrust_c[3];     /* per-rotor thrust f(w) = c0 + c1 w + c2 w^2 (N), w in rotor-speed units */
    double torque_c;        /* yaw torque per unit thrust (m) */
    double motor_tau;       /* first-order motor time constant T_m (s) */
    double rpm_min, rpm_max;/* rotor-speed range */
    double gravity;         /* m/s^2, acting along -z */
} l2f_params;

/* Reward constants of P:148-151; C_rab is a 4-vector in normalised action space (Q9). */
typedef struct {
    double C_rp, C_rq, C_rv, C_rw, C_ra;
    double C_rab[4];
    double C_rs;
} l2f_reward_weights;

/* Curriculum: stage k = floor(t / interval); each weight w_k = w_{k-1} * factor,
 * clamped at target in the direction of travel; the exploration sigma follows the same
 * scheme.  interval = 0 keeps stage 0.  C_rab is not scheduled. */
typedef struct {
    l2f_reward_weights init, target, factor;
    double sigma_init, sigma_target, sigma_factor;
    int64_t interval;
} l2f_curriculum;

typedef struct {
    uint32_t abi_version;      /* must be L2F_ABI_VERSION */
    uint32_t flags;            /* L2F_* feature flags */
    int64_t num_envs;          /* N > 0 on this device */
    uint64_t env_id_offset;    /* global id of local env 0 (sharding, Q20); offset + N <= 2^32 */
    uint64_t seed;             /* Philox key */
    int32_t action_history;    /* N_H in [0, 32] */
    int32_t max_episode_steps; /* truncation cap (Q15); 0 = none */
    double dt;                 /* integration step (s); 0.01 = 100 Hz */
    l2f_params params;         /* nominal parameters */
    double dr_lo, dr_hi;       /* DR factor range, each factor ~ U[dr_lo, dr_hi] (Q19) */
    double init_pos, init_angle, init_vel, init_angvel; /* initial-state bounds (Q17) */
    double init_rpm_lo, init_rpm_hi;
    double dist_force, dist_torque;  /* disturbance bounds, component-wise uniform (Q18) */
    double obs_sigma[4];       /* observation noise sigma for p, R, v, omega (Q8) */
    double term_pos, term_vel, term_angvel; /* termination thresholds (Q14) */
    l2f_curriculum curriculum;
} l2f_config;

/* Optional per-step outputs (device pointers; any may be NULL). */
typedef struct {
    float* obs_core;    /* [18][N]: noisy {p, R, v, omega} of the state after the step (or the
                           reset state if the episode ended and auto-reset is on), Q11 */
    float* obs_dense;   /* [N][18 + 4 N_H]: obs_core transposed + H, most recent first */
    float* reward;      /* [N] */
    uint8_t* flags;     /* [N] L2F_DONE_* bits */
    float* final_state; /* [17][N]: s' before any auto-reset */
    float* obs_critic;  /* [28][N]: privileged critic observation {p, R, v, omega, omega_m, f_r,
                           tau_r}, noise-free, of the same state as obs_core */
} l2f_step_out;

/* Actor MLP in_dim -> hidden -> hidden -> 4 (BASELINE configs[3]; Q21): ReLU hidden layers,
 * tanh output; every weight and bias an IEEE fp16 bit pattern, row-major [out][in]; layer
 * inputs are rounded to fp16, accumulation is FP32 on the tensor cores.
 * in_dim must equal 18 + 4 N_H; hidden must be 64.  Device pointers. */
typedef struct {
    const uint16_t *W1, *b1, *W2, *b2, *W3, *b3;
    int32_t in_dim, hidden;
} l2f_policy;

/* Borrowed device views into the env workspace (valid until l2f_destroy).  The caller may
 * read or overwrite them between calls (checkpoint / resume / set_state).  q is not
 * re-normalised on write (precondition ||q|| = 1).
 * Layout: structure of arrays of float4 groups plus a tail: for an array of C components,
 * components c < 4 floor(C/4) of env i are float (c/4) N 4 + 4 i + c % 4 (a warp moves each
 * group as 512 contiguous bytes, one 128-bit access per thread), and the C % 4 remaining
 * components follow as an [N][C % 4] block.  Exactly 4 C N bytes, no padding. */
typedef struct {
    float* state;      /* C = 17: [4][N][4] (p, q(w,x,y,z), v, omega, omega_m 0..2) + [N] omega_m3 */
    float* dist;       /* C = 6:  [1][N][4] (f_r world N, tau_x) + [N][2] (tau_y, tau_z) body N m */
    float* dr;         /* C = 5:  [1][N][4] (m, J_xx, J_yy, J_zz factors) + [N] thrust factor;
                          factors are 1 when DR is off */
    float* hist;       /* [N_H][N][4] ring: slot (tau mod N_H) holds the action applied at step tau */
    int32_t* hist_t0;  /* [N] first step of the current episode */
    float* hist_fill;  /* [N][4] the episode's initial history value (Q10)                      */
                       /* Logical history at step t, H[k] (k-th most recent): tau = t-1-k;
                          H[k] = hist[tau mod N_H] if tau >= hist_t0 else hist_fill.  A reset
                          writes only hist_t0 / hist_fill (O(1) bytes per env, not N_H x 16).  */
    int32_t* ep_step;  /* [N] */
    float* ep_return;  /* [N] */
    uint64_t t;        /* global step counter: the next l2f_step is step t (< 2^31) */
    int64_t num_envs;
    int32_t action_history;
} l2f_state_view;

/* ---- lifecycle ---------------------------------------------------------------------- */

/* Bytes of device workspace an env with this config needs.  Validates the config:
 * INVALID_ARGUMENT for N <= 0, N_H outside [0,32], dt <= 0, rpm_max <= rpm_min,
 * T_m <= 0, mass/inertia <= 0, offset + N > 2^32, dr_lo <= 0 or dr_lo > dr_hi, or hover
 * infeasible at the worst DR corner (4 f(rpm_max) <= m g). */
L2F_API l2f_status l2f_workspace_size(const l2f_config* cfg, size_t* bytes);

/* Creates an env over a caller-owned, 256-byte-aligned device workspace; the env's device is
 * the workspace's (cudaPointerGetAttributes), so no device argument is taken (Q38).
 * Copies cfg.  Does not touch the workspace: call l2f_reset before stepping. */
L2F_API l2f_status l2f_create(const l2f_config* cfg, void* d_workspace, size_t bytes, l2f_env** out);

/* Frees host-side resources (never the caller's workspace). */
L2F_API l2f_status l2f_destroy(l2f_env* env);

/* ---- stepping ----------------------------------------------------------------------- */

/* Resets the envs where d_mask[i] != 0 (d_mask == NULL: all envs and the episode
 * statistics), drawing initial state, disturbance, DR factors from Philox counter t
 * (Q17-Q20), filling the history (Q10) and zeroing episode counters.
 * Writes obs_core / obs_dense of the reset envs if requested (obs noise counter t). */
L2F_API l2f_status l2f_reset(l2f_env* env, const uint8_t* d_mask, const l2f_step_out* out, void* stream);

/* One environment step for all N envs.  d_actions: [4][N] in [-1,1] (clipped
 * after exploration noise).  Then t += 1.  HBM-bound; one kernel launch. */
L2F_API l2f_status l2f_step(l2f_env* env, const float* d_actions, const l2f_step_out* out, void* stream);

/* Fused rollout of T >= 1 steps in one persistent launch, state in registers.
 *  policy != NULL: actions from the actor MLP on the noisy observation (tcgen05 tensor
 *                  cores; requires N_H % 4 == 0); d_actions must be NULL.
 *  policy == NULL, d_actions != NULL: open loop, actions [T][4][N].
 *  policy == NULL, d_actions == NULL: open loop, Philox random actions U(-1,1) (stream 6).
 * d_trace: NULL or [T][K][32] floats for the K local env indices d_trace_ids[K] (device):
 *   fields 0-16 pre-step state, 17-20 raw action, 21-24 applied action, 25 reward,
 *   26 flags, 27 ep_step after the step, 28-31 zero.  Then t += T.
 * With a policy the history ring is held in fp16 on chip, so afterwards it holds q16(a'). */
L2F_API l2f_status l2f_rollout(l2f_env* env, const l2f_policy* policy, const float* d_actions,
                       int32_t T, float* d_trace, const int64_t* d_trace_ids, int32_t K,
                       void* stream);

/* Reduces the episode statistics accumulated since the last reset of the accumulators into
 * d_out[8] (FP64, fixed-order, deterministic).  reset_accumulators != 0 zeroes them. */
L2F_API l2f_status l2f_episode_stats(l2f_env* env, double* d_out, int32_t reset_accumulators, void* stream);

/* Reward recalculation over a replay buffer: rewards of M stored transitions
 * (s' [17][M], applied action a' [4][M], device) under the curriculum stage of step t
 * (P:152), into d_rewards [M].  Bitwise equal to the reward l2f_step returned for the same
 * (s', a', stage); 0 for a non-finite s' (Q26).  Uses only env's config (no env state). */
L2F_API l2f_status l2f_recompute_rewards(const l2f_env* env, uint64_t t, const float* d_next_state,
                                         const float* d_actions, int64_t m, float* d_rewards, void* stream);

/* ---- host-buffer entry points (end-to-end; synchronise the stream before returning) --- */

/* H2D of h_actions [4][N], l2f_step, D2H of the requested outputs (any may be NULL). */
L2F_API l2f_status l2f_step_host(l2f_env* env, const float* h_actions, float* h_obs_core,
                         float* h_reward, uint8_t* h_flags, void* stream);

/* H2D of a host policy (fp16 bits) into the env's workspace, l2f_rollout(T), then
 * l2f_episode_stats(reset_accumulators) D2H into h_stats[8] (may be NULL). */
L2F_API l2f_status l2f_rollout_host(l2f_env* env, const l2f_policy* h_policy, int32_t T,
                            double* h_stats, int32_t reset_accumulators, void* stream);

/* ---- Lissajous tracking evaluation (Table III) ------ */

/* Figure-eight reference p_ref(t) = [amp_x cos(2 pi t/T_c), amp_y sin(4 pi t/T_c), altitude]
 * (the paper's [cos(2 pi t/T), sin(4 pi t/T)/2, const] is amp_x = 1, amp_y = 0.5), v_ref its
 * analytic derivative, t = k dt for tracking step k (Q28). */
typedef struct {
    const float* cycle_time;  /* [N] device: cycle time T_c of each env (s, > 0); a batch can
                                 sweep T_c (Table III: 15, 5.5, 3.5 s)                      */
    double amp_x, amp_y, altitude;
    double clip_pos, clip_vel; /* setpoint-shift clipping bounds (Q29), > 0          */
    int32_t n_steps;           /* steps simulated, >= 1                                     */
    float* rmse;               /* [N] out: RMSE of p - p_ref over x, y, z (m), completed steps */
    float* rmse_xy;            /* [N] out: the same over x, y                                */
    int32_t* steps_ok;         /* [N] out: steps completed before the first termination (Q31);
                                  n_steps = the run succeeded                               */
} l2f_tracking;

/* Batched tracking of the reference by the actor with setpoint shifting: every env
 * starts at p_ref(0) at rest (q = identity, w = 0, rotors at the hover speed, history filled
 * with the hover action, no disturbance, nominal parameters; Q30); each step the actor sees
 * its observation (noise per cfg.flags) with p and v replaced by clip(p - p_ref) and
 * clip(v - v_ref) (Q29), acts deterministically (no exploration noise), the env transitions
 * (RK4), and the error p - p_ref at the new time accumulates (FP64) until the first
 * termination, which (with L2F_TERMINATION) is tested on the tracking-error state
 * (|p - p_ref|_inf, |v - v_ref|, |w| against the training bounds) or on divergence (Q31).
 * Overwrites the env state (it ends in the final tracking state with a valid history ring;
 * call l2f_reset before training again) and advances t by n_steps.  Needs a policy
 * (in_dim 18 + 4 N_H, N_H % 4 == 0).  INVALID_ARGUMENT for NULL pointers, n_steps < 1 or
 * clip bounds <= 0. */
L2F_API l2f_status l2f_track(l2f_env* env, const l2f_policy* policy, const l2f_tracking* spec, void* stream);

/* ---- batched TD3 update (Q32-Q35) ---------- */

/* TD3 hyper-parameters (S:436 defaults: gamma 0.99, tau 0.005, sigma_t 0.2, clip_t 0.5,
 * lr 3e-4 / 3e-4, Adam beta1 0.9, beta2 0.999, eps 1e-8). */
typedef struct {
    double gamma, tau, sigma_t, clip_t, lr_actor, lr_critic, beta1, beta2, eps;
} l2f_td3_hyper;

/* One replay batch per agent, device FP32, [A][B][...] row-major: actor observations o_a /
 * o_a2 [in_dim], critic observations o_c / o_c2 [28] (l2f_step_out.obs_critic layout per
 * sample), actions a [4] (as applied), rewards r, done (1 = terminal, 0 otherwise; truncation
 * is not terminal), eps [4]: standard normals of the target-policy smoothing noise (drawn
 * by the caller, e.g. torch.randn). */
typedef struct {
    const float *o_a, *o_c, *a, *r, *o_a2, *o_c2, *done, *eps;
} l2f_td3_batch;

/* Sizes: floats of one agent's parameter block and bytes of its scratch.  Block layout
 * (FP32): [actor, actor', Q1, Q2, Q1', Q2', m_actor, v_actor, m_Q1, v_Q1, m_Q2, v_Q2]; each
 * net is W1[64][in], b1[64], W2[64][64], b2[64], W3[out][64], b3[out] with the actor
 * in_dim -> 4 (ReLU, ReLU, tanh) and the critics 32 -> 1 (ReLU, ReLU, linear) on
 * concat(o_c, a).  INVALID_ARGUMENT unless 1 <= batch <= 256 and 1 <= in_dim <= 156 (the
 * paper's largest observation, N_H = 32, is 146; the bound is the kernel's shared-memory plan). */
L2F_API l2f_status l2f_td3_sizes(int32_t in_dim, int32_t batch, int64_t* block_floats,
                                 int64_t* scratch_bytes_per_agent);

/* One TD3 update of each of n_agents independent agents (one CTA each): clipped double-Q
 * target with clipped smoothing noise, both critics regressed by MSE (one Adam step each,
 * Adam step number t_critic >= 1), and if update_actor (the delayed step, every d-th call):
 * the deterministic policy gradient through the updated Q1's action input (Adam step
 * t_actor >= 1) and Polyak averaging of the three targets with tau.  d_losses [A][3] out:
 * critic 1, critic 2, actor (0 when not updated).  d_scratch: n_agents x scratch bytes,
 * caller-owned; after the call it holds the raw gradients (documented for tests: see
 * l2f_td3.cu).  All pointers device, asynchronous on `stream`. */
L2F_API l2f_status l2f_td3_update(float* d_params, int32_t n_agents, int32_t in_dim, int32_t batch,
                                  const l2f_td3_batch* b, const l2f_td3_hyper* h, int64_t t_critic,
                                  int64_t t_actor, int32_t update_actor, float* d_losses, void* d_scratch,
                                  void* stream);

/* The actor of agent `agent` of a TD3 parameter block array as the fp16 rollout policy:
 * writes W1[64][in_dim], b1[64], W2[64][64], b2[64], W3[4][64], b3[4] (fp16 bits, round to
 * nearest even) contiguously to d_out (caller-owned, 64 in_dim + 4420 halves) and fills *out
 * with pointers into it, ready for l2f_rollout / l2f_policy_forward / l2f_track -- training
 * and rollouts stay on the device.  Asynchronous on `stream`. */
L2F_API l2f_status l2f_td3_export_actor(const float* d_params, int32_t agent, int32_t in_dim, uint16_t* d_out,
                                        l2f_policy* out, void* stream);

/* ---- state access --------------------------------------------------------------------- */

L2F_API l2f_status l2f_get_state(l2f_env* env, l2f_state_view* out);
L2F_API l2f_status l2f_set_t(l2f_env* env, uint64_t t);

/* Checkpoint restore (SURVEY 8(b) set_state): asynchronously copies every non-NULL
 * array of `in` (caller-owned DEVICE buffers in the l2f_state_view layouts above) into the
 * env's workspace on `stream`, then sets the step counter to in->t.  in->num_envs and
 * in->action_history must equal the env's (INVALID_ARGUMENT otherwise; nothing copied).
 * NULL arrays keep the current contents.  q is not re-normalised (precondition ||q|| = 1).
 * Restoring a snapshot taken with l2f_get_state (copied out) resumes the run bitwise:
 * the RNG is keyed by (env id, t), not by a stateful generator. */
L2F_API l2f_status l2f_set_state(l2f_env* env, const l2f_state_view* in, void* stream);

/* Actor MLP forward on explicit observations (the same tcgen05 tile code as the rollout):
 * d_obs [N][in_dim] fp32, d_act [N][4] fp32 (tanh output, before noise). */
L2F_API l2f_status l2f_policy_forward(const l2f_policy* policy, const float* d_obs, float* d_act,
                              int64_t n, void* stream);

/* Diagnostics: writes our Philox4x32-10 output and curand_Philox4x32_10's for counters
 * (i, t, i mod 7, i mod 5), key = seed, i < n, into d_ours[n][4] / d_curand[n][4] (uint32). */
L2F_API l2f_status l2f_selftest_philox(int64_t n, uint64_t seed, uint32_t t, uint32_t* d_ours, uint32_t* d_curand,
                                       void* stream);

/* Number of kernels this library launched since load (diagnostics for the bench). */
L2F_API uint64_t l2f_launch_count(void);

L2F_API const char* l2f_last_error(void);
L2F_API int32_t l2f_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* L2F_H */
