/*
 * dog_oracle.h -- CPU ORACLE for the DS-PHD/MIB filter cycle (TEST INFRASTRUCTURE ONLY).
 *
 * This header and dog_oracle.c are the plain, slow, obviously-correct reference the CUDA path is
 * checked against.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load or call it.  The product library (libdog.so) never links or includes it,
 * and it includes nothing from the product (no shared headers, constants or helpers).
 *
 * Paper: Nuss et al., "A Random Finite Set Approach for Dynamic Occupancy Grid Maps with Real-Time
 * Application", arXiv 1605.02406 -- /root/reference/PAPER.md, cited as P:<line>.  Readings of
 * silent/ambiguous points are DESIGN.md section 3 (A-1 .. A-31, numbering from SURVEY.md 8(c)).
 */
#ifndef DOG_ORACLE_H
#define DOG_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t width, height;   /* cells; key = row*width + col (A-4)                          */
    float   cell_size;       /* metres per cell (Table I: 0.1 m)                    */
    int64_t nu;              /* persistent particles nu (Table I)                   */
    int64_t nu_b;            /* birth particles nu_b per step (Table I)      */
    float   p_s;             /* persistence probability (Eq. 39)                 */
    float   p_b;             /* birth probability (Eqs. 67-68)                 */
    float   sigma_pos;       /* m per (T/s)   (Table I; A-1 linear in T)             */
    float   sigma_vel;       /* (m/s) per (T/s) (Table I; A-1)                       */
    float   sigma_birth_vel; /* m/s (Table I)                                        */
    float   free_tau;        /* s: alpha(T) = exp(-T/free_tau) (Eq. 62; A-9)    */
    float   occ_max;         /* cap on predicted occupied mass (Eq. 17; A-7)      */
    float   v_max;           /* |v| clamp of new-borns, <= 0 disables (A-16)                */
    uint64_t seed;           /* Philox key (A-20)                                           */
} orc_params;

typedef struct orc_ctx orc_ctx;

/* Stage dumps of the last orc_step (for stage-level parity). */
enum {
    ORC_PRED_X = 1, ORC_PRED_Y, ORC_PRED_VX, ORC_PRED_VY, /* f32 [nu] predicted state, input order */
    ORC_KEY,          /* u32 [nu] cell key, C = outside (A-4, A-5)                    */
    ORC_PERM,         /* u32 [nu] stable sort: perm[j] = input index of sorted slot j  */
    ORC_OFFSETS,      /* u32 [C+1] exclusive prefix of n_c                             */
    ORC_S,            /* f32 [C] sum of predicted weights (Eq. 61)                     */
    ORC_MP,           /* f32 [C] m_p = min(S, occ_max) (Eq. 17/61)                     */
    ORC_MFP,          /* f32 [C] predicted free mass (Eq. 62)                          */
    ORC_OCC,          /* f32 [C] posterior m_O (Eq. 63)                                */
    ORC_FREE,         /* f32 [C] posterior m_F (Eq. 63)                                */
    ORC_RHO_P,        /* f32 [C] (Eq. 68)                                              */
    ORC_RHO_B,        /* f32 [C] (Eq. 67)                                              */
    ORC_RP,           /* u64 [C] fixed-point persistent mass (A-23)                   */
    ORC_RB,           /* u64 [C] fixed-point born mass, gated by m_zO > 0 (A-13, A-23) */
    ORC_NB,           /* u32 [C] birth slots per cell (A-15)                           */
    ORC_BIRTH_X, ORC_BIRTH_Y, ORC_BIRTH_VX, ORC_BIRTH_VY, /* f32 [nu_b] (A-16) */
    ORC_BIRTH_CELL,   /* u32 [nu_b] cell of each slot (C if unused)                    */
    ORC_MEAN,         /* f32 [C][2] (Eq. 81)                                           */
    ORC_COV,          /* f32 [C][3] var_x, var_y, cov_xy (Eqs. 83-84)                  */
    ORC_JOINT_IDX,    /* u32 [nu] selected joint index j(i) (Alg. 7, A-24, A-25)       */
    ORC_SCALARS,      /* u64 [8]: W, U, A, meas_bad_count, w_pred bits, w_bar bits, k, n_in */
    ORC_GFX,          /* u32 [nu] fixed-point Doppler likelihood, input order (NEXT-1, A-34) */
    ORC_GS,           /* u64 [C] its sum over the cell's members (0: no Doppler / guard)  */
    ORC_NA,           /* u32 [C] associated birth slots nu_A (A-36)                    */
    ORC_RBA           /* u64 [C] born mass of the associated set R_bA (A-36)           */
};

/* --- primitives (exported for the pins in tests/) --- */
void  orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float orc_u01(uint32_t r);            /* (r>>8) * 2^-24, in [0,1)                 */
float orc_u01_open(uint32_t r);       /* ((r>>8)|1) * 2^-24, in (0,1)             */
float orc_ln_u24(uint32_t m);         /* ln(m * 2^-24), m odd, written spec (A-20) */
void  orc_sincos_2pi_u24(uint32_t n, float* s, float* c); /* sin/cos(2 pi n 2^-24), n < 2^24 */
void  orc_box_muller(uint32_t ra, uint32_t rb, float* z0, float* z1);
void  orc_dempster(float aO, float aF, float bO, float bF, float* mO, float* mF);
void  orc_birth_split(float m_p, float m_O, float p_b, float* rho_b, float* rho_p);
/* slots: Rb[C] (u64) -> nb[C] (u32); returns total A's low 64 bits */
uint64_t orc_birth_slots(const uint64_t* Rb, int64_t C, int64_t nu_b, uint32_t* nb);
/* fixed-point exponent FX of the masses for a grid of C cells (A-23): 40 while C < 2^24 */
int orc_fx_bits(int64_t C);
/* systematic resampling on a plain weight list q[n] (u64): idx[nu] (Alg. 7, A-24) */
uint64_t orc_systematic_resample(const uint64_t* q, int64_t n, int64_t nu, uint32_t U, uint32_t* idx);
void  orc_step_scalars(const orc_params* p, float dt, float out[4]); /* Tc, s_p, s_v, alpha */

/* --- the filter --- */
int  orc_create(const orc_params* p, orc_ctx** out);
void orc_destroy(orc_ctx* h);
int  orc_set_state(orc_ctx* h, const float* x, const float* y, const float* vx, const float* vy,
                   float w_bar, const float* m_free, int64_t k);
int  orc_get_state(orc_ctx* h, float* x, float* y, float* vx, float* vy, float* w_bar,
                   float* m_free, int64_t* k);
/* meas: float[C][2] = (m_zO, m_zF) row-major; dt > 0 seconds */
int  orc_step(orc_ctx* h, const float* meas, float dt);
/* Doppler / association branch (NEXT-1; Eqs. 69-80):
 * dop[C][4] = (u_x, u_y, v_r, sd) radial unit direction, measured radial speed (m/s) and its SD;
 * pA[C] = association probability p_A in [0, 1] (0: no Doppler in the cell).  NULL: orc_step. */
int  orc_step_doppler(orc_ctx* h, const float* meas, const float* dop, const float* pA, float dt);
/* The exact PHD/MIB filter (NEXT-3; section V) with a uniform likelihood equal to the
 * clutter density (section IV-F setting): obs[C][4] = (occurred 0/1, p_TP, p_FP, unused) (A-37).
 * m_F is not used (left unchanged); occupancy readout = rho_p + rho_b, free = 1 - occupancy. */
int  orc_step_exact(orc_ctx* h, const float* obs, float dt);
int  orc_step_exact_lik(orc_ctx* h, const float* obs, const float* lik, const float* pA, float dt);
float orc_birth_mean_lik(float vr, float sd, float sigma_b);
void orc_exact_lik_cell(float S, float occ_max, float p_b, float pTP, float pFP, float pcl, float pA, uint64_t GS,
                        float gmax, uint32_t n, float vr, float sd, float sigma_b, float* rho_p, float* rho_b,
                        float* pAe, float* pi);
void orc_birth_assoc_exact(uint64_t Rb, uint32_t nb, float pi, uint32_t* nA, uint64_t* RbA);
void orc_exact_cell(float S, float occ_max, float p_b, float occurred, float pTP, float pFP, float* rho_p,
                    float* rho_b);
/* NEXT-1 primitives (exported for the pins) */
float    orc_exp_spec(float q);                                             /* e^q, q <= 0 (A-34) */
float    orc_doppler_g(float vx, float vy, float ux, float uy, float vr, float sd);   /* Eq. 69 g */
uint32_t orc_doppler_gfx(float g, float gmax);                              /* floor(g/gmax 2^31) */
uint64_t orc_doppler_Q(uint64_t Rp, float pA, uint64_t GSj, uint64_t GS, uint32_t j, uint32_t n);
void     orc_birth_assoc(uint64_t Rb, uint32_t nb, float pA, uint32_t* nA, uint64_t* RbA);
/* Ego-motion compensation (NEXT-2): scroll grid and particles by the whole-cell part of (dx, dy) plus the
 * stored residual (metres); returns -1 (nothing changed) if a shift would reach half the grid side. */
int  orc_ego_scroll(orc_ctx* h, double dx, double dy, int32_t* shift_x, int32_t* shift_y);
void orc_ego_residual(const orc_ctx* h, double* rx, double* ry);

/* Evaluation workload (NEXT-4): per-cell Mahalanobis distance of the velocity estimate
 * from v = 0 (Eq. 88), static/dynamic classification counts per threshold, and the sums behind the
 * cluster statistics (Eqs. 85-86).  A pure function of the readouts:
 *   mean[C][2], cov[C][3] (var_x, var_y, cov_xy), valid[C] (moments reported; NULL: mean or cov != 0),
 *   labels[C] (0 unlabeled, 1 static, 2 dynamic; NULL: no counts), mask[C] (cluster S; NULL: no sums),
 *   thr[n_thr] -> m[C] (f32, may be NULL), counts[n_thr][4] = (TP, FN, FP, TN) with "dynamic
 *   detection" = m >= thr, sums[5] = (|S|, sum mean_x, sum (var_x + mean_x^2), sum mean_y,
 *   sum (var_y + mean_y^2)). */
void orc_eval_cells(int64_t C, const float* mean, const float* cov, const uint8_t* valid, const uint8_t* labels,
                    const uint8_t* mask, const float* thr, int n_thr, float* m, uint64_t* counts, double* sums);
/* readouts of the last step: occ[C], free[C], mean[C][2], cov[C][3] */
int  orc_read_cells(orc_ctx* h, float* occ, float* free_mass, float* mean, float* cov);
/* copy a stage dump of the last step; returns bytes copied or <0 */
int64_t orc_get_dump(orc_ctx* h, int what, void* dst, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif
