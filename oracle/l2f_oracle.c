/*
 * l2f_oracle.c -- plain, slow, obviously-correct FP64 CPU oracle for the batched
 * quadrotor environment step of arXiv 2311.13081 ("Learning to Fly in Seconds").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2311_13081_b200/, libl2f.so) never links, loads or calls it, and this file
 * shares no code, header, table or constant generator with paper_2311_13081_b200/csrc.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets);
 *            "S:n" = /root/reference/SPEC.md line n (interface ideas only);
 *            "Qn"  = a reading of the paper listed in DESIGN.md section 3.
 *
 * Everything is FP64 except (a) the Philox integers and (b) the fp16 quantisation of the
 * actor MLP's operands, which is part of the method's definition as this build states it
 * (Q21: fp16 parameters and fp16 layer inputs, wide accumulation).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): Philox KAT vectors (Random123), fp16 rounding
 * vs numpy.float16, R(q) orthonormality/det/double cover/Rodrigues, hover derivative = 0,
 * free fall z = -g t^2/2, discrete motor-lag closed form and the 63 % step response,
 * single-axis roll/yaw torque closed forms, RK4 4th-order convergence, reward special cases
 * (P:148-151), termination edge cases, curriculum closed form, reset-distribution
 * bounds/moments, MLP vs numpy matmul on fp16-rounded operands, Lissajous reference closed
 * forms and the exact-hover tracking RMSE (sqrt(13/8) over whole cycles).
 * Parity unpinned: long free-running closed-loop MLP trajectories (checked teacher-forced and
 * by distribution only); absolute physical constants (P:21 - the paper's
 * parameter PDF is absent).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------------------ */
/* Types (the oracle's own; the Python wrapper in oracle/__init__.py mirrors them).       */
/* ------------------------------------------------------------------------------------ */

/* Quadrotor parameters.  Only m = 0.027 kg and T_m = 0.15 s are paper values
 * (P:141); the rest live in the absent supplementary PDF. */
typedef struct {
    double mass;            /* kg */
    double J[3];            /* diagonal inertia, kg m^2 */
    double rotor_pos[4][3]; /* body frame, m */
    double spin_dir[4];     /* +-1 */
    double thrust_c[3];     /* f(w) = c0 + c1 w + c2 w^2, N */
    double torque_c;        /* yaw torque per unit thrust, m */
    double motor_tau;       /* first-order motor time constant T_m, s */
    double rpm_min, rpm_max;
    double gravity;         /* m/s^2 along -z */
} or_params;

/* Reward constants C_* (P:148-151). C_rab is a 4-vector (Q9). */
typedef struct {
    double C_rp, C_rq, C_rv, C_rw, C_ra, C_rab[4], C_rs;
} or_weights;

enum {
    OR_OBS_NOISE = 1u << 0,
    OR_ACTION_NOISE = 1u << 1,
    OR_TERMINATION = 1u << 2,
    OR_AUTO_RESET = 1u << 3,
    OR_DISTURBANCE = 1u << 4,
    OR_DOMAIN_RAND = 1u << 5,
    OR_NO_ROTOR_DELAY = 1u << 6, /* ablation, Table II "Rotor Delay" */
};

enum { OR_FLAG_TERMINATED = 1, OR_FLAG_TRUNCATED = 2, OR_FLAG_DIVERGED = 4, OR_FLAG_RESET = 8 };

/* Philox streams (Q20). */
enum { OR_STREAM_ACT = 1, OR_STREAM_OBS = 2, OR_STREAM_RESET = 3, OR_STREAM_DIST = 4,
       OR_STREAM_DR = 5, OR_STREAM_RAND_ACT = 6 };

typedef struct {
    uint32_t flags;
    int32_t n_hist;            /* N_H, 0..32 */
    int32_t max_episode_steps; /* 0 = no truncation */
    int32_t pad0;
    uint64_t seed;
    double dt;                 /* 0.01 s = 100 Hz */
    or_params nominal;
    double dr_lo, dr_hi;       /* multiplicative DR range (Q19) */
    double init_pos, init_angle, init_vel, init_angvel, init_rpm_lo, init_rpm_hi; /* Q17 */
    double dist_force, dist_torque;  /* Q18 */
    double obs_sigma[4];       /* p, R, v, omega (Q8) */
    double term_pos, term_vel, term_angvel; /* Q14 */
    or_weights w_init, w_target, w_factor;  /* curriculum */
    double sigma_init, sigma_target, sigma_factor; /* exploration noise decay */
    int64_t interval;          /* curriculum interval in env steps; 0 = stage 0 forever */
} or_config;

/* One environment.  hist[k] = H[k] = the action applied k+1 steps ago (most recent first,
 * S:116); this plain shifted array is the definition, not a ring. */
typedef struct {
    double s[17];     /* p(3) q(4: w,x,y,z) v(3) omega(3) omega_m(4) */
    double dist[6];   /* f_r (world, N), tau_r (body, N m) */
    double dr[5];     /* DR factors: mass, Jxx, Jyy, Jzz, thrust scale (Q19); 1 when off */
    double hist[32][4];
    int64_t ep_step;
    double ep_return;
} or_env;

typedef struct {
    double reward;
    uint32_t flags;
    uint32_t pad;
    double a_applied[4];
    double final_s[17];     /* s' before any reset */
    double margin[3];       /* max|p|-P, |v|-V, |w|-W  (Q22) */
} or_step_out;

/* Actor MLP: in_dim -> hidden -> hidden -> 4, all parameters given as fp16 bit patterns
 * (Q21).  Row-major [out][in]. */
typedef struct {
    int32_t in_dim, hidden;
    const uint16_t *W1, *b1, *W2, *b2, *W3, *b3;
} or_policy;

/* Episode statistics. */
enum { OR_ST_EPISODES = 0, OR_ST_TERMINATED, OR_ST_TRUNCATED, OR_ST_DIVERGED, OR_ST_SUM_LEN,
       OR_ST_SUM_RET, OR_ST_SUM_RET_SQ, OR_ST_ENV_STEPS, OR_ST_LEN };

/* ------------------------------------------------------------------------------------ */
/* Counter-based RNG: Philox4x32-10 (Salmon et al. 2011, Random123).  Q20.                */
/* ------------------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k0;
        uint32_t n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* Draw block `block` of stream `stream` for env `env_id` at step counter `t` (Q20). */
static void draw_block(const or_config* cfg, uint64_t env_id, uint64_t t, uint32_t stream,
                       uint32_t block, uint32_t out[4])
{
    uint32_t ctr[4] = {(uint32_t)env_id, (uint32_t)t, stream, block};
    uint32_t key[2] = {(uint32_t)cfg->seed, (uint32_t)(cfg->seed >> 32)};
    or_philox4x32_10(ctr, key, out);
}

/* 23-bit uniform in (0,1): u = ((x >> 9) + 1/2) 2^-23 (Q20).  Every value is exactly
 * representable in fp32 (2k+1 < 2^24), so both sides of the parity test draw the same u. */
double or_uniform(uint32_t x) { return ((double)(x >> 9) + 0.5) * (1.0 / 8388608.0); }

/* Box-Muller (Q20): (x_a, x_b) -> (r cos 2 pi u2, r sin 2 pi u2), r = sqrt(-2 ln u1). */
void or_box_muller(uint32_t xa, uint32_t xb, double z[2])
{
    double u1 = or_uniform(xa), u2 = or_uniform(xb);
    double r = sqrt(-2.0 * log(u1));
    z[0] = r * cos(2.0 * M_PI * u2);
    z[1] = r * sin(2.0 * M_PI * u2);
}

/* Four standard normals from one Philox block. */
static void normals4(const uint32_t x[4], double z[4])
{
    or_box_muller(x[0], x[1], z);
    or_box_muller(x[2], x[3], z + 2);
}

/* ------------------------------------------------------------------------------------ */
/* fp16 (IEEE binary16) rounding, round-to-nearest-even (Q21).                             */
/* ------------------------------------------------------------------------------------ */
double or_q16(double x)
{
    if (isnan(x)) return x;
    double ax = fabs(x);
    if (ax >= 65520.0) return copysign(INFINITY, x); /* beyond max half 65504 + half-ulp */
    double quantum;
    if (ax < 6.103515625e-05) {           /* below 2^-14: subnormal spacing 2^-24 */
        quantum = ldexp(1.0, -24);
    } else {
        int e;
        frexp(ax, &e);                    /* ax = m 2^e, m in [0.5, 1) */
        quantum = ldexp(1.0, e - 11);     /* 11 significant bits */
    }
    return copysign(nearbyint(ax / quantum) * quantum, x); /* default mode: ties-to-even */
}

double or_half_to_double(uint16_t h)
{
    int sign = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(1024 + m), e - 25);
    return sign ? -v : v;
}

/* ------------------------------------------------------------------------------------ */
/* Rotation matrix from quaternion.  Hamilton (w,x,y,z),            */
/* world-from-body (Q4).  Row-major.                                                     */
/* ------------------------------------------------------------------------------------ */
void or_rotation(const double q[4], double R[9])
{
    double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* Per-env effective parameters: nominal scaled by DR factors (Q19). */
void or_effective_params(const or_config* cfg, const double dr[5], or_params* p)
{
    *p = cfg->nominal;
    p->mass = cfg->nominal.mass * dr[0];
    p->J[0] = cfg->nominal.J[0] * dr[1];
    p->J[1] = cfg->nominal.J[1] * dr[2];
    p->J[2] = cfg->nominal.J[2] * dr[3];
    for (int j = 0; j < 3; ++j) p->thrust_c[j] = cfg->nominal.thrust_c[j] * dr[4];
}

/* ------------------------------------------------------------------------------------ */
/* Dynamics derivative (equations as).                      */
/*   f_i = c0 + c1 w_i + c2 w_i^2  ("non-linear torque/thrust curves", Q3)           */
/*   p' = v                                                                              */
/*   q' = 1/2 q (x) (0, omega)                                                           */
/*   v' = (0,0,-g) + (R(q) (0,0,sum f) + f_r) / m                                        */
/*   omega' = J^-1 (tau - omega x J omega),                                              */
/*        tau = sum r_i x (0,0,f_i) + (0,0, c_tau sum d_i f_i) + tau_r                     */
/*   omega_m' = (u - omega_m) / T_m        (first-order motor lag)          */
/* ------------------------------------------------------------------------------------ */
void or_derivative(const or_params* P, const double s[17], const double u[4],
                   const double dist[6], double ds[17])
{
    const double* p = s; (void)p;
    const double* q = s + 3;
    const double* v = s + 7;
    const double* w = s + 10;
    const double* wm = s + 13;

    double f[4], T = 0.0;
    for (int i = 0; i < 4; ++i) {
        f[i] = P->thrust_c[0] + P->thrust_c[1] * wm[i] + P->thrust_c[2] * wm[i] * wm[i];
        T += f[i];
    }
    double tau[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 4; ++i) {
        /* r_i x (0,0,f_i) = (r_y f, -r_x f, 0) */
        tau[0] += P->rotor_pos[i][1] * f[i];
        tau[1] += -P->rotor_pos[i][0] * f[i];
        tau[2] += P->torque_c * P->spin_dir[i] * f[i];
    }
    for (int j = 0; j < 3; ++j) tau[j] += dist[3 + j];

    /* p' = v */
    ds[0] = v[0]; ds[1] = v[1]; ds[2] = v[2];
    /* q' = 1/2 q (x) (0, w)  (Hamilton product) */
    ds[3] = 0.5 * (-q[1] * w[0] - q[2] * w[1] - q[3] * w[2]);
    ds[4] = 0.5 * (q[0] * w[0] + q[2] * w[2] - q[3] * w[1]);
    ds[5] = 0.5 * (q[0] * w[1] - q[1] * w[2] + q[3] * w[0]);
    ds[6] = 0.5 * (q[0] * w[2] + q[1] * w[1] - q[2] * w[0]);
    /* v' */
    double R[9];
    or_rotation(q, R);
    for (int j = 0; j < 3; ++j) ds[7 + j] = (R[3 * j + 2] * T + dist[j]) / P->mass;
    ds[9] -= P->gravity;
    /* omega' = J^-1 (tau - omega x (J omega)) */
    double Jw[3] = {P->J[0] * w[0], P->J[1] * w[1], P->J[2] * w[2]};
    double cx = w[1] * Jw[2] - w[2] * Jw[1];
    double cy = w[2] * Jw[0] - w[0] * Jw[2];
    double cz = w[0] * Jw[1] - w[1] * Jw[0];
    ds[10] = (tau[0] - cx) / P->J[0];
    ds[11] = (tau[1] - cy) / P->J[1];
    ds[12] = (tau[2] - cz) / P->J[2];
    /* omega_m' = (u - omega_m) / T_m */
    for (int i = 0; i < 4; ++i) ds[13 + i] = (u[i] - wm[i]) / P->motor_tau;
}

/* Classical RK4 over one step h with zero-order-hold u (Q1). */
void or_rk4(const or_params* P, const double s[17], const double u[4], const double dist[6],
            double h, double out[17])
{
    double k1[17], k2[17], k3[17], k4[17], tmp[17];
    or_derivative(P, s, u, dist, k1);
    for (int i = 0; i < 17; ++i) tmp[i] = s[i] + 0.5 * h * k1[i];
    or_derivative(P, tmp, u, dist, k2);
    for (int i = 0; i < 17; ++i) tmp[i] = s[i] + 0.5 * h * k2[i];
    or_derivative(P, tmp, u, dist, k3);
    for (int i = 0; i < 17; ++i) tmp[i] = s[i] + h * k3[i];
    or_derivative(P, tmp, u, dist, k4);
    for (int i = 0; i < 17; ++i) out[i] = s[i] + h / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
}

/* Post-integration projection (Q5): renormalise q, clamp motor speeds. */
void or_project(const or_params* P, double s[17])
{
    double n = sqrt(s[3] * s[3] + s[4] * s[4] + s[5] * s[5] + s[6] * s[6]);
    for (int i = 3; i < 7; ++i) s[i] /= n;
    for (int i = 13; i < 17; ++i) s[i] = fmin(fmax(s[i], P->rpm_min), P->rpm_max);
}

/* Action map [-1,1] -> [w_min, w_max] (Q6). */
double or_action_to_rpm(const or_params* P, double a)
{
    return P->rpm_min + (a + 1.0) * 0.5 * (P->rpm_max - P->rpm_min);
}

/* ------------------------------------------------------------------------------------ */
/* Curriculum: every `interval` steps each weight is multiplied by its factor    */
/* until it reaches its target, where it stays.  The exploration noise follows the same  */
/* exponential scheme.  Stage k = floor(t / interval).                            */
/* ------------------------------------------------------------------------------------ */
static double toward(double w, double f, double target, double init)
{
    double n = w * f;
    return (init <= target) ? fmin(n, target) : fmax(n, target);
}

void or_stage(const or_config* cfg, int64_t t, or_weights* w, double* sigma_a)
{
    int64_t k = cfg->interval > 0 ? t / cfg->interval : 0;
    *w = cfg->w_init;
    double sg = cfg->sigma_init;
    const or_weights *I = &cfg->w_init, *F = &cfg->w_factor, *G = &cfg->w_target;
    for (int64_t j = 0; j < k; ++j) {
        w->C_rp = toward(w->C_rp, F->C_rp, G->C_rp, I->C_rp);
        w->C_rq = toward(w->C_rq, F->C_rq, G->C_rq, I->C_rq);
        w->C_rv = toward(w->C_rv, F->C_rv, G->C_rv, I->C_rv);
        w->C_rw = toward(w->C_rw, F->C_rw, G->C_rw, I->C_rw);
        w->C_ra = toward(w->C_ra, F->C_ra, G->C_ra, I->C_ra);
        w->C_rs = toward(w->C_rs, F->C_rs, G->C_rs, I->C_rs);
        sg = toward(sg, cfg->sigma_factor, cfg->sigma_target, cfg->sigma_init);
    }
    *sigma_a = sg;
}

/* Reward, evaluated on the post-transition state s' (Q12). */
double or_reward(const or_weights* w, const double s[17], const double a[4])
{
    const double *p = s, *q = s + 3, *v = s + 7, *om = s + 10;
    double pp = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
    double vv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    double ww = om[0] * om[0] + om[1] * om[1] + om[2] * om[2];
    double aa = 0.0;
    for (int i = 0; i < 4; ++i) aa += (a[i] - w->C_rab[i]) * (a[i] - w->C_rab[i]);
    return -w->C_rp * pp - w->C_rq * (1.0 - q[0] * q[0]) - w->C_rv * vv - w->C_rw * ww
           - w->C_ra * aa + w->C_rs;
}

/* ------------------------------------------------------------------------------------ */
/* Reset: initial state, disturbance, DR factors, history fill (Q10, Q17-Q19) */
/* ------------------------------------------------------------------------------------ */
static double uab(double a, double b, uint32_t x) { return a + (b - a) * or_uniform(x); }

void or_reset(const or_config* cfg, uint64_t env_id, uint64_t counter, or_env* e)
{
    uint32_t b0[4], b1[4], b2[4], b3[4];
    draw_block(cfg, env_id, counter, OR_STREAM_RESET, 0, b0);
    draw_block(cfg, env_id, counter, OR_STREAM_RESET, 1, b1);
    draw_block(cfg, env_id, counter, OR_STREAM_RESET, 2, b2);
    draw_block(cfg, env_id, counter, OR_STREAM_RESET, 3, b3);
    double P0 = cfg->init_pos, V0 = cfg->init_vel, W0 = cfg->init_angvel;
    /* position ~ U[-P0, P0]^3 */
    e->s[0] = uab(-P0, P0, b0[0]);
    e->s[1] = uab(-P0, P0, b0[1]);
    e->s[2] = uab(-P0, P0, b0[2]);
    /* attitude: uniform axis (cz ~ U[-1,1], phi ~ U[0, 2pi)), angle ~ U[0, theta_max] */
    double cz = uab(-1.0, 1.0, b0[3]);
    double phi = 2.0 * M_PI * or_uniform(b1[0]);
    double theta = cfg->init_angle * or_uniform(b1[1]);
    double sxy = sqrt(1.0 - cz * cz);
    double ax = sxy * cos(phi), ay = sxy * sin(phi), az = cz;
    e->s[3] = cos(0.5 * theta);
    e->s[4] = sin(0.5 * theta) * ax;
    e->s[5] = sin(0.5 * theta) * ay;
    e->s[6] = sin(0.5 * theta) * az;
    /* linear velocity ~ U[-V0, V0]^3 */
    e->s[7] = uab(-V0, V0, b1[2]);
    e->s[8] = uab(-V0, V0, b1[3]);
    e->s[9] = uab(-V0, V0, b2[0]);
    /* angular velocity ~ U[-W0, W0]^3 */
    e->s[10] = uab(-W0, W0, b2[1]);
    e->s[11] = uab(-W0, W0, b2[2]);
    e->s[12] = uab(-W0, W0, b2[3]);
    /* rotor speeds ~ U[lo, hi] */
    for (int i = 0; i < 4; ++i) e->s[13 + i] = uab(cfg->init_rpm_lo, cfg->init_rpm_hi, b3[i]);

    /* disturbance, sampled at the beginning of each episode */
    if (cfg->flags & OR_DISTURBANCE) {
        uint32_t d0[4], d1[4];
        draw_block(cfg, env_id, counter, OR_STREAM_DIST, 0, d0);
        draw_block(cfg, env_id, counter, OR_STREAM_DIST, 1, d1);
        double F = cfg->dist_force, Tq = cfg->dist_torque;
        e->dist[0] = uab(-F, F, d0[0]);
        e->dist[1] = uab(-F, F, d0[1]);
        e->dist[2] = uab(-F, F, d0[2]);
        e->dist[3] = uab(-Tq, Tq, d0[3]);
        e->dist[4] = uab(-Tq, Tq, d1[0]);
        e->dist[5] = uab(-Tq, Tq, d1[1]);
    } else {
        for (int j = 0; j < 6; ++j) e->dist[j] = 0.0;
    }
    /* domain randomisation factors, per episode (Q19; BASELINE configs[2]) */
    if (cfg->flags & OR_DOMAIN_RAND) {
        uint32_t r0[4], r1[4];
        draw_block(cfg, env_id, counter, OR_STREAM_DR, 0, r0);
        draw_block(cfg, env_id, counter, OR_STREAM_DR, 1, r1);
        e->dr[0] = uab(cfg->dr_lo, cfg->dr_hi, r0[0]);
        e->dr[1] = uab(cfg->dr_lo, cfg->dr_hi, r0[1]);
        e->dr[2] = uab(cfg->dr_lo, cfg->dr_hi, r0[2]);
        e->dr[3] = uab(cfg->dr_lo, cfg->dr_hi, r0[3]);
        e->dr[4] = uab(cfg->dr_lo, cfg->dr_hi, r1[0]);
    } else {
        for (int j = 0; j < 5; ++j) e->dr[j] = 1.0;
    }
    /* action history filled with the normalised equivalent of the initial rotor speeds (Q10) */
    const or_params* P = &cfg->nominal;
    for (int k = 0; k < 32; ++k)
        for (int i = 0; i < 4; ++i)
            e->hist[k][i] = (k < cfg->n_hist)
                ? 2.0 * (e->s[13 + i] - P->rpm_min) / (P->rpm_max - P->rpm_min) - 1.0 : 0.0;
    e->ep_step = 0;
    e->ep_return = 0.0;
}

/* ------------------------------------------------------------------------------------ */
/* Actor observation o_a = {p, R, v, omega, H}, noise on the first 18 only   */
/* (Q8).  Obs noise normal i in [0,18) is normal (i mod 4) of Philox block */
/* floor(i/4) of stream OBS at counter t (Q20).                                          */
/* ------------------------------------------------------------------------------------ */
void or_observe(const or_config* cfg, const or_env* e, uint64_t env_id, uint64_t t, double* obs)
{
    double R[9];
    or_rotation(e->s + 3, R);
    for (int j = 0; j < 3; ++j) obs[j] = e->s[j];
    for (int j = 0; j < 9; ++j) obs[3 + j] = R[j];
    for (int j = 0; j < 3; ++j) obs[12 + j] = e->s[7 + j];
    for (int j = 0; j < 3; ++j) obs[15 + j] = e->s[10 + j];
    if (cfg->flags & OR_OBS_NOISE) {
        double z[20];
        for (int b = 0; b < 5; ++b) {
            uint32_t x[4];
            draw_block(cfg, env_id, t, OR_STREAM_OBS, (uint32_t)b, x);
            normals4(x, z + 4 * b);
        }
        for (int i = 0; i < 18; ++i) {
            int grp = i < 3 ? 0 : (i < 12 ? 1 : (i < 15 ? 2 : 3));
            obs[i] += cfg->obs_sigma[grp] * z[i];
        }
    }
    for (int k = 0; k < cfg->n_hist; ++k)
        for (int i = 0; i < 4; ++i) obs[18 + 4 * k + i] = e->hist[k][i];
}

/* Privileged critic observation o_c = {p, R, v, omega, omega_m, f_r, tau_r}, 28-D,
 * ground truth without noise. */
void or_critic_observe(const or_env* e, double* obs)
{
    double R[9];
    or_rotation(e->s + 3, R);
    for (int j = 0; j < 3; ++j) obs[j] = e->s[j];
    for (int j = 0; j < 9; ++j) obs[3 + j] = R[j];
    for (int j = 0; j < 3; ++j) obs[12 + j] = e->s[7 + j];
    for (int j = 0; j < 3; ++j) obs[15 + j] = e->s[10 + j];
    for (int j = 0; j < 4; ++j) obs[18 + j] = e->s[13 + j];
    for (int j = 0; j < 3; ++j) obs[22 + j] = e->dist[j];
    for (int j = 0; j < 3; ++j) obs[25 + j] = e->dist[3 + j];
}

/* Reward recalculation of a stored transition: the reward of (s', a') under the
 * curriculum stage of step t; 0 for a non-finite s' (Q26). */
double or_recompute_reward(const or_config* cfg, int64_t t, const double s1[17], const double a[4])
{
    or_weights w;
    double sg;
    for (int i = 0; i < 17; ++i)
        if (!isfinite(s1[i])) return 0.0;
    or_stage(cfg, t, &w, &sg);
    return or_reward(&w, s1, a);
}

/* ------------------------------------------------------------------------------------ */
/* Actor MLP (architecture from BASELINE configs[3]; precision Q21).        */
/* h1 = relu(W1 q16(o) + b1); h2 = relu(W2 q16(h1) + b2); a = tanh(W3 q16(h2) + b3).      */
/* ------------------------------------------------------------------------------------ */
void or_mlp(const or_policy* pol, const double* obs, double a[4])
{
    int I = pol->in_dim, H = pol->hidden;
    double x0[256], h1[256], h2[256];
    for (int i = 0; i < I; ++i) x0[i] = or_q16(obs[i]);
    for (int j = 0; j < H; ++j) {
        double acc = or_half_to_double(pol->b1[j]);
        for (int i = 0; i < I; ++i) acc += or_half_to_double(pol->W1[j * I + i]) * x0[i];
        h1[j] = or_q16(acc > 0.0 ? acc : 0.0);
    }
    for (int j = 0; j < H; ++j) {
        double acc = or_half_to_double(pol->b2[j]);
        for (int i = 0; i < H; ++i) acc += or_half_to_double(pol->W2[j * H + i]) * h1[i];
        h2[j] = or_q16(acc > 0.0 ? acc : 0.0);
    }
    for (int j = 0; j < 4; ++j) {
        double acc = or_half_to_double(pol->b3[j]);
        for (int i = 0; i < H; ++i) acc += or_half_to_double(pol->W3[j * H + i]) * h2[i];
        a[j] = tanh(acc);
    }
}

/* Relative distance of x != 0 to the nearest fp16 rounding midpoint (SURVEY 8(c) parity test
 * 5): the midpoints around x are those of h = |q16(x)| and its two fp16 neighbours, h + u/2
 * above and h - d/2 below, where u is the spacing above h and d the spacing below it (d = u/2
 * when h is a normal power of two, where the binade changes; the subnormal spacing 2^-24 also
 * holds up to and including 2^-14). */
static double midpoint_margin(double x)
{
    double ax = fabs(x), h = fabs(or_q16(x));
    if (!(ax > 0.0) || isinf(h)) return INFINITY;
    double up, down;
    if (h < 6.103515625e-05) {
        up = down = ldexp(1.0, -24);
    } else {
        int e;
        double m = frexp(h, &e);          /* h = m 2^e, m in [0.5, 1) */
        up = ldexp(1.0, e - 11);
        down = (m == 0.5 && h > 6.103515625e-05) ? 0.5 * up : up;
    }
    double above = (h + 0.5 * up) - ax, below = h > 0.0 ? ax - (h - 0.5 * down) : INFINITY;
    return fmin(above, below) / ax;
}

/* Pre-activation of the three layers, for the "near an fp16 rounding midpoint" exclusion
 * of the teacher-forced parity test.  Returns, over every quantisation
 * point (the observation and the positive layer-1/layer-2 pre-activations), the minimum
 * relative distance to an fp16 rounding midpoint. */
double or_mlp_min_midpoint_margin(const or_policy* pol, const double* obs)
{
    int I = pol->in_dim, H = pol->hidden;
    double x0[256], h1[256], h2[256];
    double worst = INFINITY;
#define MARGIN(v)                                                                      \
    do {                                                                               \
        double _m = midpoint_margin(v);                                                \
        if (_m < worst) worst = _m;                                                    \
    } while (0)
    for (int i = 0; i < I; ++i) { MARGIN(obs[i]); x0[i] = or_q16(obs[i]); }
    for (int j = 0; j < H; ++j) {
        double acc = or_half_to_double(pol->b1[j]);
        for (int i = 0; i < I; ++i) acc += or_half_to_double(pol->W1[j * I + i]) * x0[i];
        if (acc > 0) MARGIN(acc);
        h1[j] = or_q16(acc > 0.0 ? acc : 0.0);
    }
    for (int j = 0; j < H; ++j) {
        double acc = or_half_to_double(pol->b2[j]);
        for (int i = 0; i < H; ++i) acc += or_half_to_double(pol->W2[j * H + i]) * h1[i];
        if (acc > 0) MARGIN(acc);
        h2[j] = or_q16(acc > 0.0 ? acc : 0.0);
    }
    (void)h2;
#undef MARGIN
    return worst;
}

/* ------------------------------------------------------------------------------------ */
/* One environment step s -> s' with noise, reward, termination and auto-reset            */
/* (Q7, Q11-Q16).  t is the global step counter.             */
/* ------------------------------------------------------------------------------------ */
void or_env_step(const or_config* cfg, or_env* e, uint64_t env_id, uint64_t t,
                 const double a_in[4], or_step_out* out, double* stats)
{
    or_weights w;
    double sigma_a;
    or_stage(cfg, (int64_t)t, &w, &sigma_a);

    /* 1. exploration noise + clip (Q7) */
    double a[4];
    double z[4] = {0, 0, 0, 0};
    if (cfg->flags & OR_ACTION_NOISE) {
        uint32_t x[4];
        draw_block(cfg, env_id, t, OR_STREAM_ACT, 0, x);
        normals4(x, z);
    }
    for (int i = 0; i < 4; ++i) {
        double v = a_in[i] + ((cfg->flags & OR_ACTION_NOISE) ? sigma_a * z[i] : 0.0);
        a[i] = fmin(fmax(v, -1.0), 1.0);
    }
    /* 2. action -> RPM setpoints */
    double u[4];
    for (int i = 0; i < 4; ++i) u[i] = or_action_to_rpm(&cfg->nominal, a[i]);

    /* ablation without rotor delay: the motors reach the setpoint instantly */
    if (cfg->flags & OR_NO_ROTOR_DELAY)
        for (int i = 0; i < 4; ++i) e->s[13 + i] = u[i];

    /* 3-4. RK4 + projection (Q1, Q5) */
    or_params P;
    or_effective_params(cfg, e->dr, &P);
    double s1[17];
    or_rk4(&P, e->s, u, e->dist, cfg->dt, s1);
    or_project(&P, s1);
    int diverged = 0;
    for (int i = 0; i < 17; ++i) if (!isfinite(s1[i])) diverged = 1;

    /* 5. history push, most recent first */
    for (int k = 31; k > 0; --k)
        for (int i = 0; i < 4; ++i) e->hist[k][i] = e->hist[k - 1][i];
    for (int i = 0; i < 4; ++i) e->hist[0][i] = a[i];

    /* 6. reward on s' (Q12); a diverged transition earns 0 (Q26) */
    double r = diverged ? 0.0 : or_reward(&w, s1, a);

    /* 7. termination: crash / leaving the box (Q14); truncation (Q15) */
    double pinf = fmax(fabs(s1[0]), fmax(fabs(s1[1]), fabs(s1[2])));
    double vv = s1[7] * s1[7] + s1[8] * s1[8] + s1[9] * s1[9];
    double ww = s1[10] * s1[10] + s1[11] * s1[11] + s1[12] * s1[12];
    int term = diverged;
    if (cfg->flags & OR_TERMINATION) {
        if (pinf > cfg->term_pos || vv > cfg->term_vel * cfg->term_vel ||
            ww > cfg->term_angvel * cfg->term_angvel)
            term = 1;
    }
    e->ep_step += 1;
    e->ep_return += r;
    int trunc = !term && cfg->max_episode_steps > 0 && e->ep_step >= cfg->max_episode_steps;

    memcpy(e->s, s1, sizeof(s1));
    if (out) {
        out->reward = r;
        out->flags = (term ? OR_FLAG_TERMINATED : 0) | (trunc ? OR_FLAG_TRUNCATED : 0) |
                     (diverged ? OR_FLAG_DIVERGED : 0);
        for (int i = 0; i < 4; ++i) out->a_applied[i] = a[i];
        memcpy(out->final_s, s1, sizeof(s1));
        out->margin[0] = pinf - cfg->term_pos;
        out->margin[1] = sqrt(vv) - cfg->term_vel;
        out->margin[2] = sqrt(ww) - cfg->term_angvel;
    }
    if (stats) stats[OR_ST_ENV_STEPS] += 1.0;

    /* 8. episode end: statistics + same-step auto-reset (Q16) */
    if (term || trunc) {
        if (stats) {
            stats[OR_ST_EPISODES] += 1.0;
            stats[OR_ST_TERMINATED] += term;
            stats[OR_ST_TRUNCATED] += trunc;
            stats[OR_ST_DIVERGED] += diverged;
            stats[OR_ST_SUM_LEN] += (double)e->ep_step;
            stats[OR_ST_SUM_RET] += e->ep_return;
            stats[OR_ST_SUM_RET_SQ] += e->ep_return * e->ep_return;
        }
        if (cfg->flags & OR_AUTO_RESET) {
            or_reset(cfg, env_id, t + 1, e);
            if (out) out->flags |= OR_FLAG_RESET;
        } else {
            e->ep_step = 0;
            e->ep_return = 0.0;
        }
    }
}

/* Open-loop random action (stream RAND_ACT, Q20): a_i = -1 + 2 U(x_i). */
void or_random_action(const or_config* cfg, uint64_t env_id, uint64_t t, double a[4])
{
    uint32_t x[4];
    draw_block(cfg, env_id, t, OR_STREAM_RAND_ACT, 0, x);
    for (int i = 0; i < 4; ++i) a[i] = -1.0 + 2.0 * or_uniform(x[i]);
}

/* ------------------------------------------------------------------------------------ */
/* Rollout driver: T steps for each env, envs split statically over nthreads POSIX       */
/* threads (the envs are independent).                                      */
/*   mode 0: actions[T][n][4] given; mode 1: Philox random actions; mode 2: MLP policy.  */
/* trace (optional): [T][n][OR_TRACE] doubles per env-step:                               */
/*   s_pre[17], a_raw[4], a_applied[4], reward, flags, ep_step_after                      */
/* ------------------------------------------------------------------------------------ */
#define OR_TRACE 28

typedef struct {
    const or_config* cfg;
    or_env* envs;
    const uint64_t* env_ids;
    int64_t n, lo, hi;
    uint64_t t0;
    int32_t T, mode;
    const double* actions;
    const or_policy* pol;
    double* trace;
    double stats[OR_ST_LEN];
} or_job;

static void* rollout_worker(void* arg)
{
    or_job* J = (or_job*)arg;
    const or_config* cfg = J->cfg;
    int obs_dim = 18 + 4 * cfg->n_hist;
    double* obs = (double*)malloc(sizeof(double) * (size_t)obs_dim);
    for (int64_t i = J->lo; i < J->hi; ++i) {
        or_env* e = &J->envs[i];
        for (int32_t k = 0; k < J->T; ++k) {
            uint64_t t = J->t0 + (uint64_t)k;
            double a_raw[4];
            if (J->mode == 0) {
                for (int c = 0; c < 4; ++c) a_raw[c] = J->actions[((size_t)k * J->n + i) * 4 + c];
            } else if (J->mode == 1) {
                or_random_action(cfg, J->env_ids[i], t, a_raw);
            } else {
                or_observe(cfg, e, J->env_ids[i], t, obs);
                or_mlp(J->pol, obs, a_raw);
            }
            double* tr = J->trace ? J->trace + ((size_t)k * J->n + i) * OR_TRACE : NULL;
            if (tr) {
                memcpy(tr, e->s, sizeof(double) * 17);
                memcpy(tr + 17, a_raw, sizeof(double) * 4);
            }
            or_step_out so;
            or_env_step(cfg, e, J->env_ids[i], t, a_raw, &so, J->stats);
            if (tr) {
                memcpy(tr + 21, so.a_applied, sizeof(double) * 4);
                tr[25] = so.reward;
                tr[26] = (double)so.flags;
                tr[27] = (double)e->ep_step;
            }
        }
    }
    free(obs);
    return NULL;
}

void or_rollout(const or_config* cfg, or_env* envs, const uint64_t* env_ids, int64_t n,
                uint64_t t0, int32_t T, int32_t mode, const double* actions,
                const or_policy* pol, double* trace, double* stats, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n) nthreads = (int32_t)(n > 0 ? n : 1);
    or_job* jobs = (or_job*)calloc((size_t)nthreads, sizeof(or_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int32_t w = 0; w < nthreads; ++w) {
        or_job* J = &jobs[w];
        J->cfg = cfg; J->envs = envs; J->env_ids = env_ids; J->n = n;
        J->lo = n * w / nthreads; J->hi = n * (w + 1) / nthreads;
        J->t0 = t0; J->T = T; J->mode = mode; J->actions = actions; J->pol = pol;
        J->trace = trace;
        if (nthreads > 1) pthread_create(&th[w], NULL, rollout_worker, J);
        else rollout_worker(J);
    }
    if (nthreads > 1)
        for (int32_t w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
    /* fixed-order reduction of the per-thread statistics */
    for (int32_t w = 0; w < nthreads; ++w)
        for (int j = 0; j < OR_ST_LEN; ++j) stats[j] += jobs[w].stats[j];
    free(jobs);
    free(th);
}

/* ------------------------------------------------------------------------------------ */
/* Lissajous trajectory tracking evaluation (Table III analogue).         */
/* ------------------------------------------------------------------------------------ */

/* Figure-eight reference: p(t) = [A_x cos(2 pi t/T), A_y sin(4 pi t/T), z]
 * with A_x = 1, A_y = 1/2 in the paper's formula; v(t) = dp/dt analytically (Q28). */
void or_lissajous(double t, double Tc, double ax, double ay, double z, double p[3], double v[3])
{
    double w = 2.0 * M_PI / Tc;
    p[0] = ax * cos(w * t);
    p[1] = ay * sin(2.0 * w * t);
    p[2] = z;
    v[0] = -ax * w * sin(w * t);
    v[1] = 2.0 * ay * w * cos(2.0 * w * t);
    v[2] = 0.0;
}

/* Setpoint shifting with clipping (Q29): the actor observes p - p_ref and v - v_ref,
 * each component clipped to +-clip; the rest of the observation is unchanged.  Applied to
 * the (noisy) observation vector from or_observe. */
void or_shift_observation(double* obs, const double p_ref[3], const double v_ref[3], double clip_pos,
                          double clip_vel)
{
    for (int j = 0; j < 3; ++j) {
        obs[j] = fmin(fmax(obs[j] - p_ref[j], -clip_pos), clip_pos);
        obs[12 + j] = fmin(fmax(obs[12 + j] - v_ref[j], -clip_vel), clip_vel);
    }
}

/* Hover rotor speed: 4 f(w) = m g with f(w) = c0 + c1 w + c2 w^2 (nominal parameters). */
double or_hover_rpm(const or_params* P)
{
    double c0 = P->thrust_c[0] - P->mass * P->gravity / 4.0, c1 = P->thrust_c[1], c2 = P->thrust_c[2];
    if (c2 == 0.0) return -c0 / c1;
    return (-c1 + sqrt(c1 * c1 - 4.0 * c2 * c0)) / (2.0 * c2);
}

/* One env's tracking run (Q28-Q31): start at p_ref(0) at rest (q = identity, w = 0, rotors
 * at hover, no disturbance, nominal parameters, history filled with the normalised hover
 * speed), then n_steps steps of: shifted observation (noise per cfg) -> deterministic actor
 * (pol; pol == NULL applies the exact hover action) -> env transition without exploration
 * noise -> error e_k = p_k - p_ref(k dt).  Termination (cfg TERMINATION flag) is tested on
 * the tracking-error state (p - p_ref, v - v_ref, w) with the training bounds, plus
 * divergence; the run stops accumulating at the first termination.  Outputs RMSE over the
 * completed steps (3-D and x-y) and the number of completed steps.  The Philox counter of
 * step k is t0 + k (as in a rollout). */
void or_track(const or_config* cfg_in, const or_policy* pol, uint64_t env_id, uint64_t t0, double Tc,
              double ax, double ay, double z, double clip_pos, double clip_vel, int32_t n_steps,
              double* rmse, double* rmse_xy, int32_t* steps_ok, double* pos_trace)
{
    or_config cfg = *cfg_in;
    cfg.flags &= ~(uint32_t)(OR_ACTION_NOISE | OR_AUTO_RESET | OR_DISTURBANCE | OR_DOMAIN_RAND);
    or_env e;
    memset(&e, 0, sizeof(e));
    double pr[3], vr[3];
    or_lissajous(0.0, Tc, ax, ay, z, pr, vr);
    e.s[0] = pr[0];
    e.s[1] = pr[1];
    e.s[2] = pr[2];
    e.s[3] = 1.0;
    double w_h = or_hover_rpm(&cfg.nominal);
    double a_h = 2.0 * (w_h - cfg.nominal.rpm_min) / (cfg.nominal.rpm_max - cfg.nominal.rpm_min) - 1.0;
    for (int i = 0; i < 4; ++i) e.s[13 + i] = w_h;
    for (int i = 0; i < 5; ++i) e.dr[i] = 1.0;
    for (int k = 0; k < 32; ++k)
        for (int i = 0; i < 4; ++i) e.hist[k][i] = a_h;
    int obs_dim = 18 + 4 * cfg.n_hist;
    double* obs = (double*)malloc(sizeof(double) * (size_t)obs_dim);
    double se = 0.0, sexy = 0.0;
    int32_t ok = 0;
    for (int32_t k = 0; k < n_steps; ++k) {
        uint64_t t = t0 + (uint64_t)k;
        double a[4];
        if (pol) {
            or_observe(&cfg, &e, env_id, t, obs);
            or_lissajous((double)k * cfg.dt, Tc, ax, ay, z, pr, vr);
            or_shift_observation(obs, pr, vr, clip_pos, clip_vel);
            or_mlp(pol, obs, a);
        } else {
            for (int i = 0; i < 4; ++i) a[i] = a_h;
        }
        or_step_out so;
        uint32_t flags_saved = cfg.flags;
        cfg.flags &= ~(uint32_t)OR_TERMINATION; /* tested on the error state below */
        or_env_step(&cfg, &e, env_id, t, a, &so, NULL);
        cfg.flags = flags_saved;
        or_lissajous((double)(k + 1) * cfg.dt, Tc, ax, ay, z, pr, vr);
        double ex = e.s[0] - pr[0], ey = e.s[1] - pr[1], ez = e.s[2] - pr[2];
        double dvx = e.s[7] - vr[0], dvy = e.s[8] - vr[1], dvz = e.s[9] - vr[2];
        double ww = e.s[10] * e.s[10] + e.s[11] * e.s[11] + e.s[12] * e.s[12];
        int term = (so.flags & OR_FLAG_DIVERGED) != 0;
        if (cfg.flags & OR_TERMINATION) {
            double einf = fmax(fabs(ex), fmax(fabs(ey), fabs(ez)));
            if (einf > cfg.term_pos || dvx * dvx + dvy * dvy + dvz * dvz > cfg.term_vel * cfg.term_vel ||
                ww > cfg.term_angvel * cfg.term_angvel)
                term = 1;
        }
        if (pos_trace) {
            pos_trace[3 * k + 0] = e.s[0];
            pos_trace[3 * k + 1] = e.s[1];
            pos_trace[3 * k + 2] = e.s[2];
        }
        if (term) break;
        se += ex * ex + ey * ey + ez * ez;
        sexy += ex * ex + ey * ey;
        ok = k + 1;
    }
    free(obs);
    *rmse = ok > 0 ? sqrt(se / ok) : 0.0;
    *rmse_xy = ok > 0 ? sqrt(sexy / ok) : 0.0;
    *steps_ok = ok;
}

/* ------------------------------------------------------------------------------------ */
/* TD3 update ("we use TD3" citing Fujimoto et al. 2018; */
/* DESIGN.md Q32-Q35).  Dense nets with a flat FP64 parameter layout per net:              */
/*   W1[hid][in], b1[hid], W2[hid][hid], b2[hid], W3[out][hid], b3[out];                   */
/* actor in_dim -> 64 -> 64 -> 4 (ReLU, ReLU, tanh); critics 32 -> 64 -> 64 -> 1 (ReLU,    */
/* ReLU, linear) on concat(o_c, a) with o_c the 28-D privileged observation.               */
/* ------------------------------------------------------------------------------------ */
int64_t or_net_size(int32_t in, int32_t hid, int32_t out)
{
    return (int64_t)hid * in + hid + (int64_t)hid * hid + hid + (int64_t)out * hid + out;
}

typedef struct {
    int32_t in, hid, out;
    double *W1, *b1, *W2, *b2, *W3, *b3;
} or_net;

static or_net net_view(double* p, int32_t in, int32_t hid, int32_t out)
{
    or_net n;
    n.in = in; n.hid = hid; n.out = out;
    n.W1 = p; p += (size_t)hid * in;
    n.b1 = p; p += hid;
    n.W2 = p; p += (size_t)hid * hid;
    n.b2 = p; p += hid;
    n.W3 = p; p += (size_t)out * hid;
    n.b3 = p;
    return n;
}

/* y = f3(W3 relu(W2 relu(W1 x + b1) + b2) + b3), f3 = tanh or identity; caches h1, h2 */
static void net_forward(const or_net* n, const double* x, double* h1, double* h2, double* y, int tanh_out)
{
    for (int j = 0; j < n->hid; ++j) {
        double acc = n->b1[j];
        for (int i = 0; i < n->in; ++i) acc += n->W1[(size_t)j * n->in + i] * x[i];
        h1[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < n->hid; ++j) {
        double acc = n->b2[j];
        for (int i = 0; i < n->hid; ++i) acc += n->W2[(size_t)j * n->hid + i] * h1[i];
        h2[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int o = 0; o < n->out; ++o) {
        double acc = n->b3[o];
        for (int i = 0; i < n->hid; ++i) acc += n->W3[(size_t)o * n->hid + i] * h2[i];
        y[o] = tanh_out ? tanh(acc) : acc;
    }
}

/* Backpropagation of dL/dy through the net: accumulates dL/dtheta into g (same layout) and
 * writes dL/dx (if dx != NULL).  ReLU'(0) = 0. */
static void net_backward(const or_net* n, const double* x, const double* h1, const double* h2, const double* y,
                         int tanh_out, const double* dy, or_net* g, double* dx)
{
    double d3[8], d2[256], d1[256];
    for (int o = 0; o < n->out; ++o) d3[o] = tanh_out ? dy[o] * (1.0 - y[o] * y[o]) : dy[o];
    for (int o = 0; o < n->out; ++o) {
        g->b3[o] += d3[o];
        for (int i = 0; i < n->hid; ++i) g->W3[(size_t)o * n->hid + i] += d3[o] * h2[i];
    }
    for (int j = 0; j < n->hid; ++j) {
        double acc = 0.0;
        for (int o = 0; o < n->out; ++o) acc += n->W3[(size_t)o * n->hid + j] * d3[o];
        d2[j] = h2[j] > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < n->hid; ++j) {
        g->b2[j] += d2[j];
        for (int i = 0; i < n->hid; ++i) g->W2[(size_t)j * n->hid + i] += d2[j] * h1[i];
    }
    for (int i = 0; i < n->hid; ++i) {
        double acc = 0.0;
        for (int j = 0; j < n->hid; ++j) acc += n->W2[(size_t)j * n->hid + i] * d2[j];
        d1[i] = h1[i] > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < n->hid; ++j) {
        g->b1[j] += d1[j];
        for (int i = 0; i < n->in; ++i) g->W1[(size_t)j * n->in + i] += d1[j] * x[i];
    }
    if (dx)
        for (int i = 0; i < n->in; ++i) {
            double acc = 0.0;
            for (int j = 0; j < n->hid; ++j) acc += n->W1[(size_t)j * n->in + i] * d1[j];
            dx[i] = acc;
        }
}

typedef struct {
    double gamma, tau, sigma_t, clip_t, lr_actor, lr_critic, beta1, beta2, eps;
} or_td3_hyper;

/* Adam (Kingma & Ba 2015) step t >= 1 on n parameters. */
static void adam(double* th, double* m, double* v, const double* g, int64_t n, int64_t t, double lr,
                 const or_td3_hyper* h)
{
    double c1 = 1.0 - pow(h->beta1, (double)t), c2 = 1.0 - pow(h->beta2, (double)t);
    for (int64_t k = 0; k < n; ++k) {
        m[k] = h->beta1 * m[k] + (1.0 - h->beta1) * g[k];
        v[k] = h->beta2 * v[k] + (1.0 - h->beta2) * g[k] * g[k];
        th[k] -= lr * (m[k] / c1) / (sqrt(v[k] / c2) + h->eps);
    }
}

/* One TD3 update of one agent (Q32-Q35).  P = [actor, actor', Q1, Q2, Q1', Q2', m_actor,
 * v_actor, m_Q1, v_Q1, m_Q2, v_Q2] (flat FP64).  Batch arrays are [B][...]; eps [B][4] are
 * the standard normals of the target-policy smoothing noise (drawn by the caller).  t_critic
 * / t_actor: the Adam step numbers of this update (>= 1).  losses[3] = critic 1, critic 2,
 * actor (0 when the actor is not updated).  grads (optional, for tests): the raw gradients
 * [Q1, Q2, actor] before Adam. */
void or_td3_update(double* P, int32_t in_dim, int32_t B, const double* o_a, const double* o_c, const double* a,
                   const double* r, const double* o_a2, const double* o_c2, const double* done,
                   const double* eps, const or_td3_hyper* h, int64_t t_critic, int64_t t_actor,
                   int32_t update_actor, double* losses, double* grads)
{
    const int32_t H = 64, CI = 32;
    const int64_t na = or_net_size(in_dim, H, 4), nc = or_net_size(CI, H, 1);
    double* pa = P;
    double* pa_t = pa + na;
    double* pc[2] = {pa_t + na, pa_t + na + nc};
    double* pc_t[2] = {pc[1] + nc, pc[1] + 2 * nc};
    double* m_a = pc_t[1] + nc;
    double* v_a = m_a + na;
    double* m_c[2] = {v_a + na, v_a + na + 2 * nc};
    double* v_c[2] = {v_a + na + nc, v_a + na + 3 * nc};
    or_net actor = net_view(pa, in_dim, H, 4), actor_t = net_view(pa_t, in_dim, H, 4);
    or_net Q[2] = {net_view(pc[0], CI, H, 1), net_view(pc[1], CI, H, 1)};
    or_net Qt[2] = {net_view(pc_t[0], CI, H, 1), net_view(pc_t[1], CI, H, 1)};
    double h1[64], h2[64], out[4], x[CI];
    double* y = (double*)malloc(sizeof(double) * (size_t)B);
    /* 1. target: smoothed target action, clipped double-Q */
    for (int32_t s = 0; s < B; ++s) {
        double at[4];
        net_forward(&actor_t, o_a2 + (size_t)s * in_dim, h1, h2, at, 1);
        for (int k = 0; k < 4; ++k) {
            double nz = h->sigma_t * eps[(size_t)s * 4 + k];
            nz = fmin(fmax(nz, -h->clip_t), h->clip_t);
            at[k] = fmin(fmax(at[k] + nz, -1.0), 1.0);
        }
        for (int k = 0; k < 28; ++k) x[k] = o_c2[(size_t)s * 28 + k];
        for (int k = 0; k < 4; ++k) x[28 + k] = at[k];
        double q1, q2;
        net_forward(&Qt[0], x, h1, h2, &q1, 0);
        net_forward(&Qt[1], x, h1, h2, &q2, 0);
        y[s] = r[s] + h->gamma * (1.0 - done[s]) * fmin(q1, q2);
    }
    /* 2. critics: mean squared error to y, one Adam step each */
    double* g = (double*)calloc((size_t)(na > nc ? na : nc), sizeof(double));
    for (int c = 0; c < 2; ++c) {
        memset(g, 0, sizeof(double) * (size_t)nc);
        or_net gn = net_view(g, CI, H, 1);
        double loss = 0.0;
        for (int32_t s = 0; s < B; ++s) {
            for (int k = 0; k < 28; ++k) x[k] = o_c[(size_t)s * 28 + k];
            for (int k = 0; k < 4; ++k) x[28 + k] = a[(size_t)s * 4 + k];
            double q;
            net_forward(&Q[c], x, h1, h2, &q, 0);
            loss += (q - y[s]) * (q - y[s]) / B;
            double dq = 2.0 * (q - y[s]) / B;
            net_backward(&Q[c], x, h1, h2, &q, 0, &dq, &gn, NULL);
        }
        if (grads) memcpy(grads + (size_t)c * nc, g, sizeof(double) * (size_t)nc);
        adam(pc[c], m_c[c], v_c[c], g, nc, t_critic, h->lr_critic, h);
        losses[c] = loss;
    }
    losses[2] = 0.0;
    if (update_actor) {
        /* 3. actor: maximise Q1(o_c, pi(o_a)) with the updated Q1 (deterministic policy
         *    gradient through the critic's action input), one Adam step */
        memset(g, 0, sizeof(double) * (size_t)na);
        or_net gn = net_view(g, in_dim, H, 4);
        double* gq = (double*)calloc((size_t)nc, sizeof(double));
        or_net gqn = net_view(gq, CI, H, 1);  /* scratch: Q1's own gradient is discarded */
        double ah1[64], ah2[64], loss = 0.0;
        for (int32_t s = 0; s < B; ++s) {
            const double* xa = o_a + (size_t)s * in_dim;
            net_forward(&actor, xa, ah1, ah2, out, 1);
            for (int k = 0; k < 28; ++k) x[k] = o_c[(size_t)s * 28 + k];
            for (int k = 0; k < 4; ++k) x[28 + k] = out[k];
            double q, dq = -1.0 / B, dx[CI];
            net_forward(&Q[0], x, h1, h2, &q, 0);
            loss += -q / B;
            net_backward(&Q[0], x, h1, h2, &q, 0, &dq, &gqn, dx);
            net_backward(&actor, xa, ah1, ah2, out, 1, dx + 28, &gn, NULL);
        }
        free(gq);
        if (grads) memcpy(grads + 2 * (size_t)nc, g, sizeof(double) * (size_t)na);
        adam(pa, m_a, v_a, g, na, t_actor, h->lr_actor, h);
        losses[2] = loss;
        /* 4. Polyak averaging of all three targets (on the delayed step, as TD3 does) */
        for (int64_t k = 0; k < na; ++k) pa_t[k] = h->tau * pa[k] + (1.0 - h->tau) * pa_t[k];
        for (int c = 0; c < 2; ++c)
            for (int64_t k = 0; k < nc; ++k) pc_t[c][k] = h->tau * pc[c][k] + (1.0 - h->tau) * pc_t[c][k];
    }
    free(g);
    free(y);
}

/* Size checks for the Python mirror. */
int64_t or_sizeof_config(void) { return (int64_t)sizeof(or_config); }
int64_t or_sizeof_env(void) { return (int64_t)sizeof(or_env); }
int64_t or_sizeof_step_out(void) { return (int64_t)sizeof(or_step_out); }
