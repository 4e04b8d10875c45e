/*
 * dog_oracle.c -- CPU ORACLE of one DS-PHD/MIB filter cycle (TEST INFRASTRUCTURE ONLY).
 *
 * Plain, single-threaded, slow on purpose.  It follows the paper's cycle step by step (PAPER.md
 * section VI, and the seven stages of section VII) in plain form:
 * direct per-cell sums instead of scans, a particle-level CDF with binary search, fp64 where a
 * quantity is a real-valued sum.  Only tests/, __graft_entry__.smoke() and bench.py's reference leg
 * may use it.  It shares no code with the CUDA path (paper_1605_02406_b200/csrc).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC (A-21: no contraction,
 * IEEE single precision via SSE2, every fused multiply-add is an explicit fmaf()).
 *
 * Pinning: every function below is pinned by tests/test_oracle_*.py against paper/SPEC worked
 * examples, closed forms or brute force.  Parity unpinned: the Box-Muller
 * output distribution is pinned only statistically (the paper fixes no generator).
 */
#include "dog_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ======================================================================================
 * Random numbers (A-20).  The paper pre-samples cuRAND arrays; the
 * reading adopted here is a counter-based Philox4x32-10 stream keyed by (seed) with counter
 * (index, k_lo, stage, k_hi), so any implementation can reproduce each draw.
 * Philox4x32-10 written from its definition (Salmon et al., SC'11): 10 rounds, multipliers
 * 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85.
 * ====================================================================================== */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw(const orc_ctx* h, uint32_t index, int64_t k, uint32_t stage, uint32_t r[4]);

/* u(r) = (r>>8) 2^-24 in [0,1) and u°(r) = ((r>>8)|1) 2^-24 in (0,1): exact in f32 (A-20). */
float orc_u01(uint32_t r)      { return (float)(r >> 8) * 0x1p-24f; }
float orc_u01_open(uint32_t r) { return (float)((r >> 8) | 1u) * 0x1p-24f; }

/* ln(m 2^-24) for odd m in [1, 2^24): the written f32 spec of DESIGN.md 3.1 (A-20 option i).
 * Integer range reduction m = f 2^e, f in [sqrt(2)/2, sqrt(2)]; ln f = 2 atanh(s), s = (f-1)/(f+1),
 * odd series to s^13; result (e-24) ln2 + ln f with ln2 split hi/lo.  Only IEEE-correctly-rounded
 * operations (+, -, *, /, fmaf) are used, so any IEEE implementation gets the same bits. */
float orc_ln_u24(uint32_t m)
{
    int e = 31 - __builtin_clz(m);                 /* floor(log2 m), m >= 1 */
    float f = ldexpf((float)m, -e);                /* exact, f in [1,2) */
    if (f > 0x1.6a09e6p+0f) { f = f * 0.5f; e = e + 1; }
    float s = (f - 1.0f) / (f + 1.0f);
    float z = s * s;
    float t = 0x1.3b13b2p-3f;                      /* 2/13 */
    t = fmaf(t, z, 0x1.745d18p-3f);                /* 2/11 */
    t = fmaf(t, z, 0x1.c71c72p-3f);                /* 2/9  */
    t = fmaf(t, z, 0x1.24924ap-2f);                /* 2/7  */
    t = fmaf(t, z, 0x1.99999ap-2f);                /* 2/5  */
    t = fmaf(t, z, 0x1.555556p-1f);                /* 2/3  */
    float sz = s * z;
    float lnf = fmaf(sz, t, s + s);
    float n = (float)(e - 24);
    float r = fmaf(n, 0x1.7f7d1cp-20f, lnf);       /* ln2 lo */
    r = fmaf(n, 0x1.62e4p-1f, r);                  /* ln2 hi */
    return r;
}

/* sin/cos(2 pi n 2^-24), n in [0, 2^24): quadrant q = round(4 n 2^-24) by integer arithmetic,
 * x = (n - q 2^22) 2^-24 in [-1/8, 1/8) exactly, Taylor polynomials of sin(2 pi x) / cos(2 pi x)
 * with f32-rounded coefficients (2pi)^k/k!, then the quadrant rotation. */
void orc_sincos_2pi_u24(uint32_t n, float* s_out, float* c_out)
{
    uint32_t q = (n + (1u << 21)) >> 22;           /* 0..4 */
    int32_t rem = (int32_t)n - (int32_t)(q << 22); /* [-2^21, 2^21) */
    float x = (float)rem * 0x1p-24f;
    float z = x * x;
    float ps = -0x1.e30750p+3f;                    /* S11 */
    ps = fmaf(ps, z, 0x1.507834p+5f);              /* S9  */
    ps = fmaf(ps, z, -0x1.32d2ccp+6f);             /* S7  */
    ps = fmaf(ps, z, 0x1.466bc6p+6f);              /* S5  */
    ps = fmaf(ps, z, -0x1.4abbcep+5f);             /* S3  */
    ps = fmaf(ps, z, 0x1.921fb6p+2f);              /* S1 = 2 pi */
    float sv = x * ps;
    float pc = 0x1.f9d38ap+2f;                     /* C12 */
    pc = fmaf(pc, z, -0x1.a6d1f2p+4f);             /* C10 */
    pc = fmaf(pc, z, 0x1.e1f506p+5f);              /* C8  */
    pc = fmaf(pc, z, -0x1.55d3c8p+6f);             /* C6  */
    pc = fmaf(pc, z, 0x1.03c1f0p+6f);              /* C4  */
    pc = fmaf(pc, z, -0x1.3bd3ccp+4f);             /* C2  */
    float cv = fmaf(pc, z, 1.0f);
    switch (q & 3u) {
    case 0:  *s_out = sv;  *c_out = cv;  break;
    case 1:  *s_out = cv;  *c_out = -sv; break;
    case 2:  *s_out = -sv; *c_out = -cv; break;
    default: *s_out = -cv; *c_out = sv;  break;
    }
}

/* Box-Muller pair: (rho cos 2 pi u(rb), rho sin 2 pi u(rb)), rho = sqrt(-2 ln u°(ra)). */
void orc_box_muller(uint32_t ra, uint32_t rb, float* z0, float* z1)
{
    float l = orc_ln_u24((ra >> 8) | 1u);
    float rho = sqrtf(-2.0f * l);
    float s, c;
    orc_sincos_2pi_u24(rb >> 8, &s, &c);
    *z0 = rho * c;
    *z1 = rho * s;
}

/* exp(q) for q <= 0 -- DESIGN.md A-34 "exp spec": q < -87 -> 0 (no subnormals); otherwise
 * k = rint(q log2 e), r = (q - k ln2_hi) - k ln2_lo (two fma), e^r = 1 + r + r^2 P(r) with the cephes
 * expf coefficients (fma Horner), times 2^k (exact power of two).  IEEE single operations only. */
float orc_exp_spec(float q)
{
    if (!(q >= -87.0f)) return 0.0f;
    if (q > 0.0f) q = 0.0f;
    float kf = rintf(q * 1.44269504088896341f);
    float r = fmaf(-kf, 0.693359375f, q);
    r = fmaf(-kf, -2.12194440e-4f, r);
    float z = r * r;
    float y = 1.9875691500e-4f;
    y = fmaf(y, r, 1.3981999507e-3f);
    y = fmaf(y, r, 8.3334519073e-3f);
    y = fmaf(y, r, 4.1665795894e-2f);
    y = fmaf(y, r, 1.6666665459e-1f);
    y = fmaf(y, r, 5.0000001201e-1f);
    y = fmaf(y, z, r);
    y = y + 1.0f;
    int k = (int)kf;                       /* -126 <= k <= 0 here */
    uint32_t bits = (uint32_t)(127 + k) << 23;
    float scale; memcpy(&scale, &bits, 4);
    return y * scale;
}

/* Doppler likelihood g(z|x) of a predicted velocity (NEXT-1; Eq. 69):
 * Gaussian density of e = v . u - v_r with SD sd, in this operation order (A-34):
 * e = fma(vx, ux, vy*uy) - v_r; t = e / sd; g = exp_spec((t*t) * -0.5) / (sd * sqrt(2 pi)). */
float orc_doppler_g(float vx, float vy, float ux, float uy, float vr, float sd)
{
    float e = fmaf(vx, ux, vy * uy) - vr;
    float t = e / sd;
    float q = (t * t) * -0.5f;
    return orc_exp_spec(q) / (sd * 2.50662827463100050f);
}

/* Fixed-point likelihood of a member relative to the largest likelihood g_max of its cell (A-34):
 * gfx = floor((g / g_max) 2^31), f32 division then an exact power-of-two scale, so 0 <= gfx <= 2^31.
 * mu_A in Eq. 72 makes the weights invariant to a common scale of g, so the fractions
 * gfx_j / sum gfx are Eqs. 71-72's g_j / sum g up to a relative quantum of 2^-31 of the cell's largest
 * member; the sums stay exact integers (order-free).  g_max = 0 (every member's g underflowed in f32)
 * gives 0: the sum(w~) = 0 guard of SPEC S:253. */
uint32_t orc_doppler_gfx(float g, float gmax)
{
    const float big = 0x1.fffffep+127f;                    /* inf -> FLT_MAX so the ratio stays defined */
    float gc = g < big ? g : big, mc = gmax < big ? gmax : big;
    if (!(gc > 0.0f) || !(mc > 0.0f)) return 0u;
    float r = gc / mc;                                     /* <= 1: gc <= mc */
    return (uint32_t)(r * 2147483648.0f);
}

/* Cumulative weight fraction of member j of n in a Doppler cell (Eqs. 71-73 with p_A > 0, A-35):
 * G_j = p_A GS_j / GS + (1 - p_A) j / n in fp64 (one fma); Q_j = floor(R_p G_j).  G_0 = 0, G_n = 1
 * exactly, and G is nondecreasing in j, so the members' weights Q_{j+1} - Q_j sum to R_p exactly. */
uint64_t orc_doppler_Q(uint64_t Rp, float pA, uint64_t GSj, uint64_t GS, uint32_t j, uint32_t n)
{
    double pa = (double)pA;
    double a = (double)GSj / (double)GS;
    double b = (1.0 - pa) * ((double)j / (double)n);
    double G = fma(pa, a, b);
    return (uint64_t)((double)Rp * G);
}

/* Split of a cell's nb birth slots and born mass into the associated (A) and unassociated (A-bar)
 * sets (Eqs. 74-80; A-36): nu_A = floor(p_A nb + 1/2) (round half up), R_bA =
 * floor(R_b p_A) in fp64 (0 if nu_A = 0, R_b if nu_A = nb). */
void orc_birth_assoc(uint64_t Rb, uint32_t nb, float pA, uint32_t* nA, uint64_t* RbA)
{
    uint32_t na = (uint32_t)floor((double)pA * (double)nb + 0.5);
    if (na > nb) na = nb;
    uint64_t ra = (uint64_t)((double)Rb * (double)pA);
    if (na == 0) ra = 0;
    else if (na == nb) ra = Rb;
    *nA = na; *RbA = ra;
}

/* ======================================================================================
 * Dempster's rule on {O, F, Omega} (Eq. 63 `eq:DS_comb`; A-10) in the canonical
 * operation order of DESIGN.md 3.2.  Total conflict (1-K <= 0) returns the measurement BBA.
 * ====================================================================================== */
void orc_dempster(float aO, float aF, float bO, float bF, float* mO, float* mF)
{
    float aW = (1.0f - aO) - aF;
    float bW = (1.0f - bO) - bF;
    float K = aO * bF + aF * bO;
    float oneK = 1.0f - K;
    if (oneK <= 0.0f) { *mO = bO; *mF = bF; return; }
    *mO = (aO * bO + (aO * bW + aW * bO)) / oneK;   /* symmetric order: bitwise a(+)b == b(+)a */
    *mF = (aF * bF + (aF * bW + aW * bF)) / oneK;
}

/* Birth split, Eqs. 67-68 (A-11: Eq. 66's right-hand side read as the predicted m_p). */
void orc_birth_split(float m_p, float m_O, float p_b, float* rho_b, float* rho_p)
{
    float q = p_b * (1.0f - m_p);
    float den = m_p + q;
    float rb = den > 0.0f ? (m_O * q) / den : 0.0f;
    *rho_b = rb;
    *rho_p = m_O - rb;
}

/* Fixed-point exponent of the masses (A-23): 40 bits per unit of mass while C < 2^24; beyond, 63 minus
 * the bit length of C, so that a total over all cells (each holding at most 1 + 2^-24 units of mass after
 * rounding) stays below 2^64. */
int orc_fx_bits(int64_t C)
{
    int bits = 0;                                  /* bit length of C */
    while (bits < 62 && ((int64_t)1 << bits) <= C) ++bits;
    return bits <= 24 ? 40 : 63 - bits;
}

/* Fixed point fx(m) = floor(max(m,0) 2^FX) (A-23): exact in fp64 (a power-of-two scale). */
static uint64_t fxq(double scale, float m)
{
    if (!(m > 0.0f)) return 0;
    return (uint64_t)((double)m * scale);
}

/* Birth slot allocation (Alg. 5 lines 2-3; A-14, A-15): cumulative nearest rounding
 * of the born-mass CDF to exactly nu_b slots: s_c = floor((2 nu_b A_c + A) / (2A)). */
uint64_t orc_birth_slots(const uint64_t* Rb, int64_t C, int64_t nu_b, uint32_t* nb)
{
    u128 A = 0;
    for (int64_t c = 0; c < C; ++c) A += Rb[c];
    if (A == 0 || nu_b == 0) {
        for (int64_t c = 0; c < C; ++c) nb[c] = 0;
        return (uint64_t)A;
    }
    u128 Ac = 0, s_prev = 0;
    for (int64_t c = 0; c < C; ++c) {
        Ac += Rb[c];
        u128 s = ((u128)2 * (u128)nu_b * Ac + A) / ((u128)2 * A);
        nb[c] = (uint32_t)(s - s_prev);
        s_prev = s;
    }
    return (uint64_t)A;
}

/* Systematic resampling on an explicit weight list (Alg. 7; A-24):
 * CDF_j = inclusive prefix of q; t_i = floor((i 2^32 + U) W / (nu 2^32));
 * idx[i] = min{ j : CDF_j > t_i } found by plain binary search.  Returns W. */
uint64_t orc_systematic_resample(const uint64_t* q, int64_t n, int64_t nu, uint32_t U, uint32_t* idx)
{
    uint64_t* cdf = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint64_t));
    uint64_t acc = 0;
    for (int64_t j = 0; j < n; ++j) { acc += q[j]; cdf[j] = acc; }
    uint64_t W = acc;
    if (W > 0) {
        for (int64_t i = 0; i < nu; ++i) {
            u128 num = (((u128)(uint64_t)i << 32) + (u128)U) * (u128)W;
            uint64_t t = (uint64_t)(num / (((u128)(uint64_t)nu) << 32));
            int64_t lo = 0, hi = n - 1;            /* smallest j with cdf[j] > t */
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (cdf[mid] > t) hi = mid; else lo = mid + 1;
            }
            idx[i] = (uint32_t)lo;
        }
    }
    free(cdf);
    return W;
}

/* Per-step scalars (c.1): computed once in fp64 from the f32 parameters and rounded to f32. */
void orc_step_scalars(const orc_params* p, float dt, float out[4])
{
    double T = (double)dt;
    out[0] = (float)(T / (double)p->cell_size);                         /* Tc  */
    out[1] = (float)(((double)p->sigma_pos * T) / (double)p->cell_size); /* s_p */
    out[2] = (float)((double)p->sigma_vel * T);                         /* s_v */
    out[3] = (float)exp(-(T / (double)p->free_tau));                    /* alpha(T) (A-9) */
}

/* ======================================================================================
 * The filter state S_k (A-19, A-3): nu particles (x, y in cell units; vx, vy in m/s) in canonical
 * order, one uniform weight w_bar (Eq. 57 makes all resampled weights equal), m_F per cell, step k.
 * ====================================================================================== */
#define SENTINEL_POS (-1073741824.0f)   /* -2^30 cells: outside any grid (A-5, A-19) */

struct orc_ctx {
    orc_params p;
    int64_t C;
    float *x, *y, *vx, *vy;  /* [nu] */
    float w_bar;
    float* m_free;           /* [C] */
    int64_t k;
    /* dumps of the last step */
    float *px, *py, *pvx, *pvy;
    uint32_t *key, *perm, *offsets;
    float *S, *mp, *mfp, *occ, *fre, *rho_p, *rho_b;
    uint64_t *Rp, *Rb;
    uint32_t* nb;
    float *bx, *by, *bvx, *bvy;
    uint32_t* bcell;
    float *mean, *cov;
    uint32_t* jidx;
    uint32_t* gfx;           /* [nu] fixed-point Doppler likelihood of each predicted particle (NEXT-1) */
    uint64_t* GS;            /* [C] its sum over the cell's members                            */
    uint32_t* nA;            /* [C] associated birth slots (NEXT-1)                            */
    uint64_t* RbA;           /* [C] born mass of the associated set                            */
    float* gmaxc;            /* [C] the cell's largest member likelihood (A-34)                */
    float* pe;               /* [C] association weight of the members' split: p_A (NEXT-1) or
                                    the effective pAe of the exact filter with a likelihood (A-38) */
    float* pic;              /* [C] associated share of the births (A-38)                      */
    double fx, fx_inv;       /* 2^FX and 2^-FX: fixed-point scale of the masses (orc_fx_bits)  */
    uint64_t scal[8];
    double res_x, res_y;     /* ego-motion residual, metres (NEXT-2) */
};

static void draw(const orc_ctx* h, uint32_t index, int64_t k, uint32_t stage, uint32_t r[4])
{
    uint32_t ctr[4] = { index, (uint32_t)(uint64_t)k, stage, (uint32_t)((uint64_t)k >> 32) };
    uint32_t key[2] = { (uint32_t)h->p.seed, (uint32_t)(h->p.seed >> 32) };
    orc_philox4x32_10(ctr, key, r);
}

static void* xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }

int orc_create(const orc_params* p, orc_ctx** out)
{
    if (!p || !out || p->width <= 0 || p->height <= 0 || p->nu < 1 || p->nu_b < 0) return -1;
    orc_ctx* h = (orc_ctx*)xcalloc(1, sizeof(orc_ctx));
    h->p = *p;
    int64_t C = (int64_t)p->width * p->height, nu = p->nu, nb = p->nu_b;
    h->C = C;
    h->fx = ldexp(1.0, orc_fx_bits(C));
    h->fx_inv = ldexp(1.0, -orc_fx_bits(C));
    h->x = xcalloc(nu, 4); h->y = xcalloc(nu, 4); h->vx = xcalloc(nu, 4); h->vy = xcalloc(nu, 4);
    for (int64_t i = 0; i < nu; ++i) { h->x[i] = SENTINEL_POS; h->y[i] = SENTINEL_POS; }
    h->m_free = xcalloc(C, 4);
    h->w_bar = 0.0f; h->k = 0;
    h->px = xcalloc(nu, 4); h->py = xcalloc(nu, 4); h->pvx = xcalloc(nu, 4); h->pvy = xcalloc(nu, 4);
    h->key = xcalloc(nu, 4); h->perm = xcalloc(nu, 4); h->offsets = xcalloc(C + 1, 4);
    h->S = xcalloc(C, 4); h->mp = xcalloc(C, 4); h->mfp = xcalloc(C, 4); h->occ = xcalloc(C, 4);
    h->fre = xcalloc(C, 4); h->rho_p = xcalloc(C, 4); h->rho_b = xcalloc(C, 4);
    h->Rp = xcalloc(C, 8); h->Rb = xcalloc(C, 8); h->nb = xcalloc(C, 4);
    h->bx = xcalloc(nb, 4); h->by = xcalloc(nb, 4); h->bvx = xcalloc(nb, 4); h->bvy = xcalloc(nb, 4);
    h->bcell = xcalloc(nb, 4);
    h->mean = xcalloc(2 * C, 4); h->cov = xcalloc(3 * C, 4);
    h->jidx = xcalloc(nu, 4);
    h->gfx = xcalloc(nu, 4); h->GS = xcalloc(C, 8); h->nA = xcalloc(C, 4); h->RbA = xcalloc(C, 8);
    h->gmaxc = xcalloc(C, 4); h->pe = xcalloc(C, 4); h->pic = xcalloc(C, 4);
    *out = h;
    return 0;
}

void orc_destroy(orc_ctx* h)
{
    if (!h) return;
    void* ptrs[] = { h->x, h->y, h->vx, h->vy, h->m_free, h->px, h->py, h->pvx, h->pvy, h->key,
                     h->perm, h->offsets, h->S, h->mp, h->mfp, h->occ, h->fre, h->rho_p, h->rho_b,
                     h->Rp, h->Rb, h->nb, h->bx, h->by, h->bvx, h->bvy, h->bcell, h->mean, h->cov,
                     h->jidx, h->gfx, h->GS, h->nA, h->RbA, h->gmaxc, h->pe, h->pic };
    for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) free(ptrs[i]);
    free(h);
}

int orc_set_state(orc_ctx* h, const float* x, const float* y, const float* vx, const float* vy,
                  float w_bar, const float* m_free, int64_t k)
{
    int64_t nu = h->p.nu;
    memcpy(h->x, x, nu * 4); memcpy(h->y, y, nu * 4);
    memcpy(h->vx, vx, nu * 4); memcpy(h->vy, vy, nu * 4);
    memcpy(h->m_free, m_free, h->C * 4);
    h->w_bar = w_bar; h->k = k;
    return 0;
}

int orc_get_state(orc_ctx* h, float* x, float* y, float* vx, float* vy, float* w_bar,
                  float* m_free, int64_t* k)
{
    int64_t nu = h->p.nu;
    if (x) memcpy(x, h->x, nu * 4);
    if (y) memcpy(y, h->y, nu * 4);
    if (vx) memcpy(vx, h->vx, nu * 4);
    if (vy) memcpy(vy, h->vy, nu * 4);
    if (m_free) memcpy(m_free, h->m_free, h->C * 4);
    if (w_bar) *w_bar = h->w_bar;
    if (k) *k = h->k;
    return 0;
}

/* qsort comparator on (key, input index): a stable sort by key (A-6). */
typedef struct { uint32_t key, idx; } kv_t;
static int cmp_kv(const void* a, const void* b)
{
    const kv_t* u = (const kv_t*)a; const kv_t* v = (const kv_t*)b;
    if (u->key != v->key) return u->key < v->key ? -1 : 1;
    return u->idx < v->idx ? -1 : (u->idx > v->idx);
}

int orc_step(orc_ctx* h, const float* meas, float dt)
{
    return orc_step_doppler(h, meas, NULL, NULL, dt);
}

/* One cycle with the Doppler / association branch (NEXT-1).  dop[C][4] = (u_x, u_y, v_r, sd): unit
 * radial direction, measured radial speed (m/s), its SD; pA[C] = association probability p_A (0: the
 * cell has no Doppler measurement).  dop == NULL or pA == NULL: no cell has one (orc_step). */
static int step_impl(orc_ctx* h, const float* meas, const float* obs, const float* dop, const float* pA, float dt);

int orc_step_doppler(orc_ctx* h, const float* meas, const float* dop, const float* pA, float dt)
{
    return step_impl(h, meas, NULL, dop, pA, dt);
}

/* The exact PHD/MIB filter (NEXT-3; section V) for a uniform single-object likelihood equal
 * to the clutter density (the setting of the section IV-F proposition): the cycle of
 * orc_step with the Bernoulli update of Eqs. (38)-(42) in place of Dempster's rule (A-37).
 * obs[C][4] = (occurred, p_TP, p_FP, unused): a measurement occurred in the cell (1) or not (0),
 * its true- and false-positive probabilities. */
int orc_step_exact(orc_ctx* h, const float* obs, float dt)
{
    return step_impl(h, NULL, obs, NULL, NULL, dt);
}

/* The exact PHD/MIB filter with a single-object likelihood (NEXT-3 general form; Eqs. 38, 49-52; A-38):
 * obs[C][4] = (occurred, p_TP, p_FP, p_cl) -- the 4th value is the clutter density at the measurement;
 * lik[C][4] = (u_x, u_y, v_r, sd): the measurement's radial-velocity likelihood g(z|x) = N(v.u - v_r;
 * 0, sd^2) (the spatial likelihood of NEXT-1, Eq. 69); pA[C] = association probability.  Cells with
 * p_A = 0 or no measurement take the uniform-likelihood update of orc_step_exact. */
int orc_step_exact_lik(orc_ctx* h, const float* obs, const float* lik, const float* pA, float dt)
{
    return step_impl(h, NULL, obs, lik, pA, dt);
}

/* Cell update of the exact filter (A-37): r_p+ = min(S, occ_max) (Eq. 31 with the truncation of
 * P:938-939), r_b+ = p_B (1 - r_p+) (Eq. 32); r+ = r_p+ + r_b+; the common weight factor
 * f = p_TP / (p_FP (1 - r+) + p_TP r+) if a measurement occurred (Eqs. 38-40; the uniform likelihood
 * g_A = p_cl cancels), else (1 - p_TP) / ((1 - p_FP)(1 - r+) + (1 - p_TP) r+) (Eq. 41); rho_p = r_p+ f,
 * rho_b = r_b+ f (Eq. 42: their sum is the posterior occupancy).  f32, in this order. */
void orc_exact_cell(float S, float occ_max, float p_b, float occurred, float pTP, float pFP, float* rho_p,
                    float* rho_b)
{
    float rpp = fminf(S, occ_max);
    float rbp = p_b * (1.0f - rpp);
    float rplus = rpp + rbp;
    float rbar = 1.0f - rplus;
    float num, den;
    if (occurred > 0.0f) { num = pTP; den = pFP * rbar + pTP * rplus; }
    else { num = 1.0f - pTP; den = (1.0f - pFP) * rbar + (1.0f - pTP) * rplus; }
    float f = den > 0.0f ? num / den : 0.0f;
    *rho_p = rpp * f;
    *rho_b = rbp * f;
}

/* Expected single-object likelihood of a new-born object under the birth prior v ~ N(0, sigma_B^2 I)
 * (A-38): the radial component v.u is N(0, sigma_B^2), so E[N(v.u - v_r; 0, sd^2)] = N(v_r; 0, s^2) with
 * s^2 = sd^2 + sigma_B^2 -- evaluated like orc_doppler_g (exp spec, f32, this order). */
float orc_birth_mean_lik(float vr, float sd, float sigma_b)
{
    float s = sqrtf(sd * sd + sigma_b * sigma_b);
    float t = vr / s;
    float q = (t * t) * -0.5f;
    return orc_exp_spec(q) / (s * 2.50662827463100050f);
}

/* Cell update of the exact filter with a single-object likelihood (NEXT-3; Eqs. 49-52, P:973-1004;
 * multi-object likelihood Eq. 38; A-38), for a cell where a measurement occurred:
 *   g_A(z|x) = p_A g(z|x) + (1 - p_A) p_cl                               (the bracket of Eq. 38)
 *   persistent: sum_i w~_i = p_TP r_p+ gbar_p, gbar_p = (p_A Sg + n (1 - p_A) p_cl) / n, Sg = sum_i g_i
 *               = GS 2^-31 g_max (the members' likelihoods in the fixed point of A-34)
 *   new-born:   sum_i w~_i = p_TP r_b+ gbar_b, gbar_b = p_A E_b[g] + (1 - p_A) p_cl (orc_birth_mean_lik)
 *   mu = p_FP p_cl (1 - r+) + p_TP r_p+ gbar_p + p_TP r_b+ gbar_b        (Eq. 51)
 *   rho_p = p_TP r_p+ gbar_p / mu, rho_b = p_TP r_b+ gbar_b / mu (f32)   (Eqs. 50, 52)
 * r_p+, r_b+, r+ as orc_exact_cell (f32); the sums in fp64 in the written order.  Also returned: the
 * effective association weight of the members' split pAe = p_A Sg / (p_A Sg + n (1 - p_A) p_cl), so
 * that member j's share of rho_p is the Doppler Q_j form (orc_doppler_Q with pAe, A-35) of
 * g_A(z|x_j) / sum_i g_A(z|x_i); and the associated share of the births pi = p_A E_b[g] / gbar_b. */
void orc_exact_lik_cell(float S, float occ_max, float p_b, float pTP, float pFP, float pcl, float pA, uint64_t GS,
                        float gmax, uint32_t n, float vr, float sd, float sigma_b, float* rho_p, float* rho_b,
                        float* pAe, float* pi)
{
    float rpp = fminf(S, occ_max);
    float rbp = p_b * (1.0f - rpp);
    float rplus = rpp + rbp;
    float rbar = 1.0f - rplus;
    double pa = (double)pA, cl = (double)pcl;
    double Sg = ((double)GS * 0x1p-31) * (double)gmax;
    double gA_sum = pa * Sg + ((double)n * (1.0 - pa)) * cl;          /* sum over the members of g_A */
    double gp = n ? gA_sum / (double)n : 0.0;
    double Eb = (double)orc_birth_mean_lik(vr, sd, sigma_b);
    double gb = pa * Eb + (1.0 - pa) * cl;
    double num_p = ((double)pTP * (double)rpp) * gp;
    double num_b = ((double)pTP * (double)rbp) * gb;
    double mu = (((double)pFP * cl) * (double)rbar + num_p) + num_b;
    *rho_p = mu > 0.0 ? (float)(num_p / mu) : 0.0f;
    *rho_b = mu > 0.0 ? (float)(num_b / mu) : 0.0f;
    *pAe = gA_sum > 0.0 ? (float)((pa * Sg) / gA_sum) : 0.0f;
    *pi = gb > 0.0 ? (float)((pa * Eb) / gb) : 0.0f;
}

/* Associated births of the exact filter with a likelihood (A-38): nu_A = floor(pi nb + 1/2) of the nb
 * slots draw the radial component from the posterior given the measurement, the rest from the prior;
 * all slots share R_b evenly (one weight for the whole birth set), i.e. R_bA = nu_A floor(R_b / nb) +
 * min(nu_A, R_b mod nb) -- the first nu_A slots' part of the single even split. */
void orc_birth_assoc_exact(uint64_t Rb, uint32_t nb, float pi, uint32_t* nA, uint64_t* RbA)
{
    uint32_t na = (uint32_t)floor((double)pi * (double)nb + 0.5);
    if (na > nb) na = nb;
    uint64_t bb = nb ? Rb / nb : 0, rb = nb ? Rb % nb : 0;
    *nA = na;
    *RbA = (uint64_t)na * bb + (na < rb ? na : rb);
}

static int step_impl(orc_ctx* h, const float* meas, const float* obs, const float* dop, const float* pA, float dt)
{
    const orc_params* P = &h->p;
    const int64_t W = P->width, H = P->height, C = h->C, nu = P->nu, nu_b = P->nu_b;
    const int64_t k = h->k;
    if (!(dt > 0.0f)) return -1;
    float sc[4];
    orc_step_scalars(P, dt, sc);
    const float Tc = sc[0], s_p = sc[1], s_v = sc[2], alpha = sc[3];
    const float Wf = (float)W, Hf = (float)H;

    /* ---- O1 Predict (Alg. 1; Eq. 14; Eq. 39; A-1..A-5) ---- */
    const float w_pred = P->p_s * h->w_bar;
    for (int64_t i = 0; i < nu; ++i) {
        uint32_t r[4];
        draw(h, (uint32_t)i, k, 1u, r);
        float n0, n1, n2, n3;
        orc_box_muller(r[0], r[1], &n0, &n1);
        orc_box_muller(r[2], r[3], &n2, &n3);
        float x = h->x[i], y = h->y[i], vx = h->vx[i], vy = h->vy[i];
        /* positions move with the OLD velocity (A-2): p' = p + T v + xi_p, v' = v + xi_v */
        float xn = fmaf(s_p, n0, fmaf(vx, Tc, x));
        float yn = fmaf(s_p, n1, fmaf(vy, Tc, y));
        float vxn = fmaf(s_v, n2, vx);
        float vyn = fmaf(s_v, n3, vy);
        h->px[i] = xn; h->py[i] = yn; h->pvx[i] = vxn; h->pvy[i] = vyn;
        int inside = (xn >= 0.0f) && (xn < Wf) && (yn >= 0.0f) && (yn < Hf);
        h->key[i] = inside ? (uint32_t)((int64_t)yn * W + (int64_t)xn) : (uint32_t)C;
    }

    /* ---- O2 Assign: stable sort by cell key (Alg. 2; A-6) ---- */
    kv_t* kv = (kv_t*)xcalloc(nu, sizeof(kv_t));
    for (int64_t i = 0; i < nu; ++i) { kv[i].key = h->key[i]; kv[i].idx = (uint32_t)i; }
    qsort(kv, (size_t)nu, sizeof(kv_t), cmp_kv);
    for (int64_t j = 0; j < nu; ++j) h->perm[j] = kv[j].idx;
    uint32_t* count = (uint32_t*)xcalloc(C + 1, 4);
    for (int64_t i = 0; i < nu; ++i) count[h->key[i]]++;
    h->offsets[0] = 0;
    for (int64_t c = 0; c < C; ++c) h->offsets[c + 1] = h->offsets[c] + count[c];
    free(kv);

    /* ---- the members' likelihoods in cells with one (NEXT-1 Doppler; NEXT-3 with a likelihood: only
     *      where a measurement occurred): g from orc_doppler_g, the cell's largest g_max, the fixed point
     *      gfx relative to it (A-34) and its sum GS -- before the cell update, which needs GS (A-38) ---- */
#define LIK_CELL(c) (dop && pA && pA[c] > 0.0f && (!obs || obs[4 * (c)] > 0.0f))
    for (int64_t i = 0; i < nu; ++i) h->gfx[i] = 0u;
    for (int64_t c = 0; c < C; ++c) {
        uint32_t a = h->offsets[c], b = h->offsets[c + 1];
        h->GS[c] = 0; h->gmaxc[c] = 0.0f; h->pe[c] = 0.0f; h->pic[c] = 0.0f;
        if (!LIK_CELL(c)) continue;
        h->pe[c] = pA[c];
        const float* d = dop + 4 * c;
        float gmax = 0.0f;                                     /* the cell's largest likelihood (A-34) */
        for (uint32_t j = a; j < b; ++j) {
            uint32_t i = h->perm[j];
            float g = orc_doppler_g(h->pvx[i], h->pvy[i], d[0], d[1], d[2], d[3]);
            if (g > gmax) gmax = g;
        }
        uint64_t gs = 0;
        for (uint32_t j = a; j < b; ++j) {
            uint32_t i = h->perm[j];
            h->gfx[i] = orc_doppler_gfx(orc_doppler_g(h->pvx[i], h->pvy[i], d[0], d[1], d[2], d[3]), gmax);
            gs += h->gfx[i];
        }
        h->GS[c] = gs;
        h->gmaxc[c] = gmax;
    }

    /* ---- O3 Cells (Alg. 3; Eqs. 61-63, 67-68; A-7..A-13, A-22, A-23, A-27) ---- */
    uint64_t bad = 0;
    for (int64_t c = 0; c < C && obs; ++c) {                  /* exact PHD/MIB (NEXT-3, A-37) */
        uint32_t a = h->offsets[c], b = h->offsets[c + 1];
        double sum = 0.0;                                      /* Eq. 31: sum of predicted weights */
        for (uint32_t j = a; j < b; ++j) sum += (double)w_pred;
        float S = (float)sum;
        const float* ob = obs + 4 * c;
        float rp, rb;
        if (LIK_CELL(c)) {                                     /* a measurement with a likelihood (A-38) */
            const float* d = dop + 4 * c;
            orc_exact_lik_cell(S, P->occ_max, P->p_b, ob[1], ob[2], ob[3], pA[c], h->GS[c], h->gmaxc[c], b - a,
                               d[2], d[3], P->sigma_birth_vel, &rp, &rb, &h->pe[c], &h->pic[c]);
        } else {
            orc_exact_cell(S, P->occ_max, P->p_b, ob[0], ob[1], ob[2], &rp, &rb);
        }
        h->S[c] = S; h->mp[c] = fminf(S, P->occ_max); h->mfp[c] = 0.0f;
        h->occ[c] = rp + rb; h->fre[c] = 1.0f - (rp + rb); h->rho_p[c] = rp; h->rho_b[c] = rb;
        h->Rp[c] = (b > a) ? fxq(h->fx, rp) : 0;                     /* A-23 */
        h->Rb[c] = fxq(h->fx, rb);                                   /* births wherever r_b > 0 */
    }
    for (int64_t c = 0; c < C && !obs; ++c) {
        uint32_t a = h->offsets[c], b = h->offsets[c + 1];
        double sum = 0.0;                                      /* Eq. 61: sum of predicted weights */
        for (uint32_t j = a; j < b; ++j) sum += (double)w_pred;
        float S = (float)sum;
        float m_p = fminf(S, P->occ_max);                      /* Eq. 17 cap (A-7) */
        float m_fp = fminf(alpha * h->m_free[c], 1.0f - m_p);  /* Eq. 62 */
        float zO = meas[2 * c], zF = meas[2 * c + 1];
        if (!(zO >= 0.0f) || !(zF >= 0.0f) || !(zO + zF <= 1.0f + 1e-6f)) { bad++; zO = 0.0f; zF = 0.0f; }
        float mO, mF;
        orc_dempster(m_p, m_fp, zO, zF, &mO, &mF);             /* Eq. 63 */
        float rb, rp;
        orc_birth_split(m_p, mO, P->p_b, &rb, &rp);            /* Eqs. 67-68 */
        h->S[c] = S; h->mp[c] = m_p; h->mfp[c] = m_fp;
        h->occ[c] = mO; h->fre[c] = mF; h->rho_p[c] = rp; h->rho_b[c] = rb;
        h->m_free[c] = mF;                                     /* Alg. 3 store_values */
        h->Rp[c] = (b > a) ? fxq(h->fx, rp) : 0;                     /* A-23 */
        h->Rb[c] = (zO > 0.0f) ? fxq(h->fx, rb) : 0;                 /* P:1197 gate (A-13) */
    }

    /* ---- O4 Persistent update (Alg. 4; Eqs. 69-73) and
     *      O6 Moments (Alg. 6; Eqs. 81-84; A-18) ----
     * Cells without Doppler (p_A = 0, g = 1): every member has w = mu_Abar w_pred (Eq. 71).  Doppler
     * cells (p_A > 0, NEXT-1): w~ = g w_pred (Eq. 69) with g from orc_doppler_g, held as fixed-point
     * gfx relative to the cell's largest g (orc_doppler_gfx, A-34); the members' fixed-point weights
     * are the differences of Q_j (orc_doppler_Q, A-35), and the moments weight each member by
     * q_j / R_p.  Sum of gfx = 0 (no member compatible with the
     * measurement): the mu_A term is dropped -- the cell is treated as p_A = 0.
     * (gfx and GS were computed before the cell update; h->pe holds the split's association weight.) */
    for (int64_t c = 0; c < C; ++c) {
        uint32_t a = h->offsets[c], b = h->offsets[c + 1];
        float* mean = h->mean + 2 * c; float* cov = h->cov + 3 * c;
        mean[0] = mean[1] = 0.0f; cov[0] = cov[1] = cov[2] = 0.0f;
        float rp = h->rho_p[c], S = h->S[c];
        if (b == a || !(rp > 0.0f) || !(S > 0.0f)) continue;
        double Mx = 0, My = 0, Mxx = 0, Myy = 0, Mxy = 0, rd;
        if (h->GS[c] > 0) {                                    /* Doppler cell: weights q_j / R_p */
            const uint32_t n = b - a;
            const uint64_t Rp = h->Rp[c], GS = h->GS[c];
            if (Rp == 0) continue;
            uint64_t gsj = 0, Qj = 0;
            for (uint32_t j = 0; j < n; ++j) {
                uint32_t i = h->perm[a + j];
                gsj += h->gfx[i];
                uint64_t Qn = orc_doppler_Q(Rp, h->pe[c], gsj, GS, j + 1, n);
                double wd = (double)(Qn - Qj) * h->fx_inv, vx = (double)h->pvx[i], vy = (double)h->pvy[i];
                Mx += wd * vx; My += wd * vy;
                Mxx += wd * vx * vx; Myy += wd * vy * vy; Mxy += wd * vx * vy;
                Qj = Qn;
            }
            rd = (double)Rp * h->fx_inv;
        } else {
            for (uint32_t j = a; j < b; ++j) {
                uint32_t i = h->perm[j];
                float w = (rp / S) * w_pred;                   /* Eq. 71: w = mu_Abar w_pred */
                double wd = (double)w, vx = (double)h->pvx[i], vy = (double)h->pvy[i];
                Mx += wd * vx; My += wd * vy;
                Mxx += wd * vx * vx; Myy += wd * vy * vy; Mxy += wd * vx * vy;
            }
            rd = (double)rp;
        }
        double mx = Mx / rd, my = My / rd;
        mean[0] = (float)mx; mean[1] = (float)my;
        cov[0] = (float)(Mxx / rd - mx * mx);
        cov[1] = (float)(Myy / rd - my * my);
        cov[2] = (float)(Mxy / rd - mx * my);
    }

    /* ---- O5 Births (Alg. 5; Eqs. 74-80; A-14..A-17, A-36) ----
     * Slot r of cell c: r < nu_A -> associated set (NEXT-1): velocity from p(x|z), radial component
     * v_r + sd n0 along u, tangential sigma_B n1 along u_perp = (-u_y, u_x); otherwise the birth prior
     * N(0, sigma_B^2) per axis.  Positions uniform in the cell for both. */
    uint64_t A = orc_birth_slots(h->Rb, C, nu_b, h->nb);
    for (int64_t j = 0; j < nu_b; ++j) {
        h->bx[j] = h->by[j] = h->bvx[j] = h->bvy[j] = 0.0f; h->bcell[j] = (uint32_t)C;
    }
    for (int64_t c = 0; c < C; ++c) {
        h->nA[c] = 0; h->RbA[c] = 0;
        if (LIK_CELL(c) && h->nb[c] > 0) {
            if (obs) orc_birth_assoc_exact(h->Rb[c], h->nb[c], h->pic[c], &h->nA[c], &h->RbA[c]);   /* A-38 */
            else orc_birth_assoc(h->Rb[c], h->nb[c], pA[c], &h->nA[c], &h->RbA[c]);               /* A-36 */
        }
    }
    {
        int64_t j = 0;
        for (int64_t c = 0; c < C; ++c) {
            int64_t col = c % W, row = c / W;
            for (uint32_t r = 0; r < h->nb[c]; ++r, ++j) {
                uint32_t R[4];
                draw(h, (uint32_t)j, k, 2u, R);
                float colf = (float)col, rowf = (float)row;
                float bxv = colf + orc_u01(R[0]);
                float byv = rowf + orc_u01(R[1]);
                if (bxv >= colf + 1.0f) bxv = nextafterf(colf + 1.0f, 0.0f);
                if (byv >= rowf + 1.0f) byv = nextafterf(rowf + 1.0f, 0.0f);
                float n0, n1;
                orc_box_muller(R[2], R[3], &n0, &n1);
                float bvx, bvy;
                if (r < h->nA[c] && obs) {                     /* exact filter: the posterior given z (A-38) */
                    const float* d = dop + 4 * c;
                    const float sb2 = P->sigma_birth_vel * P->sigma_birth_vel, sd2 = d[3] * d[3];
                    const float mu_r = (d[2] * sb2) / (sb2 + sd2);
                    const float s_r = (P->sigma_birth_vel * d[3]) / sqrtf(sb2 + sd2);
                    float sr = fmaf(s_r, n0, mu_r);            /* radial speed */
                    float st = P->sigma_birth_vel * n1;        /* tangential speed */
                    bvx = fmaf(sr, d[0], -(st * d[1]));
                    bvy = fmaf(sr, d[1], st * d[0]);
                } else if (r < h->nA[c]) {                     /* associated: p(x | z), Eq. 74 */
                    const float* d = dop + 4 * c;
                    float sr = fmaf(d[3], n0, d[2]);           /* radial speed */
                    float st = P->sigma_birth_vel * n1;        /* tangential speed */
                    bvx = fmaf(sr, d[0], -(st * d[1]));
                    bvy = fmaf(sr, d[1], st * d[0]);
                } else {                                       /* unassociated: birth prior, Eq. 76 */
                    bvx = P->sigma_birth_vel * n0; bvy = P->sigma_birth_vel * n1;
                }
                if (P->v_max > 0.0f) {
                    bvx = fminf(fmaxf(bvx, -P->v_max), P->v_max);
                    bvy = fminf(fmaxf(bvy, -P->v_max), P->v_max);
                }
                h->bx[j] = bxv; h->by[j] = byv; h->bvx[j] = bvx; h->bvy[j] = bvy;
                h->bcell[j] = (uint32_t)c;
            }
        }
    }

    /* ---- O7 Resample (Alg. 7; Eq. 57; A-24..A-26) ----
     * Joint list in cell-interleaved order (A-25): for each cell its persistent particles (sorted
     * order) then its birth slots.  Resampling weight of each member: the cell's fixed-point mass
     * split evenly, the first (R mod n) members one unit heavier (A-23). */
    int64_t n_in = h->offsets[C];
    int64_t n_joint = n_in + nu_b;
    uint64_t* q = (uint64_t*)xcalloc(n_joint, 8);
    int64_t* src = (int64_t*)xcalloc(n_joint, 8);      /* >=0: input particle, <0: -1-slot */
    {
        int64_t jj = 0, slot = 0;
        for (int64_t c = 0; c < C; ++c) {
            uint32_t a = h->offsets[c], b = h->offsets[c + 1], n = b - a;
            if (h->GS[c] > 0) {                                /* Doppler cell (A-35) */
                uint64_t gsj = 0, Qj = 0;
                for (uint32_t r = 0; r < n; ++r, ++jj) {
                    gsj += h->gfx[h->perm[a + r]];
                    uint64_t Qn = orc_doppler_Q(h->Rp[c], h->pe[c], gsj, h->GS[c], r + 1, n);
                    q[jj] = Qn - Qj;
                    Qj = Qn;
                    src[jj] = h->perm[a + r];
                }
            } else {
                for (uint32_t r = 0; r < n; ++r, ++jj) {
                    q[jj] = h->Rp[c] / n + ((uint64_t)r < h->Rp[c] % n ? 1u : 0u);
                    src[jj] = h->perm[a + r];
                }
            }
            /* births: the associated set first (nu_A slots sharing R_bA), then the unassociated set */
            uint32_t m = h->nb[c], mA = h->nA[c], mB = m - mA;
            uint64_t RA = h->RbA[c], RB = h->Rb[c] - RA;
            for (uint32_t r = 0; r < m; ++r, ++jj, ++slot) {
                if (r < mA) q[jj] = RA / mA + ((uint64_t)r < RA % mA ? 1u : 0u);
                else q[jj] = RB / mB + ((uint64_t)(r - mA) < RB % mB ? 1u : 0u);
                src[jj] = -1 - slot;
            }
        }
        n_joint = jj;
    }
    uint32_t R3[4];
    draw(h, 0u, k, 3u, R3);
    uint32_t U = R3[0];
    uint64_t Wt = orc_systematic_resample(q, n_joint, nu, U, h->jidx);
    if (Wt == 0) {
        for (int64_t i = 0; i < nu; ++i) {
            h->x[i] = SENTINEL_POS; h->y[i] = SENTINEL_POS; h->vx[i] = 0.0f; h->vy[i] = 0.0f;
            h->jidx[i] = 0xFFFFFFFFu;
        }
        h->w_bar = 0.0f;
    } else {
        for (int64_t i = 0; i < nu; ++i) {
            int64_t s = src[h->jidx[i]];
            if (s >= 0) {
                h->x[i] = h->px[s]; h->y[i] = h->py[s]; h->vx[i] = h->pvx[s]; h->vy[i] = h->pvy[s];
            } else {
                int64_t b = -1 - s;
                h->x[i] = h->bx[b]; h->y[i] = h->by[b]; h->vx[i] = h->bvx[b]; h->vy[i] = h->bvy[b];
            }
        }
        h->w_bar = (float)((double)Wt * h->fx_inv / (double)nu);   /* Eq. 57 */
    }
    free(q); free(src); free(count);

    h->scal[0] = Wt; h->scal[1] = U; h->scal[2] = A; h->scal[3] = bad;
    uint32_t wb; memcpy(&wb, &w_pred, 4); h->scal[4] = wb;
    memcpy(&wb, &h->w_bar, 4); h->scal[5] = wb;
    h->scal[6] = (uint64_t)k; h->scal[7] = (uint64_t)n_in;
    h->k = k + 1;
    return bad ? 1 : 0;
}

int orc_read_cells(orc_ctx* h, float* occ, float* free_mass, float* mean, float* cov)
{
    int64_t C = h->C;
    if (occ) memcpy(occ, h->occ, C * 4);
    if (free_mass) memcpy(free_mass, h->fre, C * 4);
    if (mean) memcpy(mean, h->mean, 2 * C * 4);
    if (cov) memcpy(cov, h->cov, 3 * C * 4);
    return 0;
}

int64_t orc_get_dump(orc_ctx* h, int what, void* dst, size_t bytes)
{
    int64_t C = h->C, nu = h->p.nu, nb = h->p.nu_b;
    const void* src = NULL; size_t n = 0;
    switch (what) {
    case ORC_PRED_X: src = h->px; n = nu * 4; break;
    case ORC_PRED_Y: src = h->py; n = nu * 4; break;
    case ORC_PRED_VX: src = h->pvx; n = nu * 4; break;
    case ORC_PRED_VY: src = h->pvy; n = nu * 4; break;
    case ORC_KEY: src = h->key; n = nu * 4; break;
    case ORC_PERM: src = h->perm; n = nu * 4; break;
    case ORC_OFFSETS: src = h->offsets; n = (C + 1) * 4; break;
    case ORC_S: src = h->S; n = C * 4; break;
    case ORC_MP: src = h->mp; n = C * 4; break;
    case ORC_MFP: src = h->mfp; n = C * 4; break;
    case ORC_OCC: src = h->occ; n = C * 4; break;
    case ORC_FREE: src = h->fre; n = C * 4; break;
    case ORC_RHO_P: src = h->rho_p; n = C * 4; break;
    case ORC_RHO_B: src = h->rho_b; n = C * 4; break;
    case ORC_RP: src = h->Rp; n = C * 8; break;
    case ORC_RB: src = h->Rb; n = C * 8; break;
    case ORC_NB: src = h->nb; n = C * 4; break;
    case ORC_BIRTH_X: src = h->bx; n = nb * 4; break;
    case ORC_BIRTH_Y: src = h->by; n = nb * 4; break;
    case ORC_BIRTH_VX: src = h->bvx; n = nb * 4; break;
    case ORC_BIRTH_VY: src = h->bvy; n = nb * 4; break;
    case ORC_BIRTH_CELL: src = h->bcell; n = nb * 4; break;
    case ORC_MEAN: src = h->mean; n = 2 * C * 4; break;
    case ORC_COV: src = h->cov; n = 3 * C * 4; break;
    case ORC_JOINT_IDX: src = h->jidx; n = nu * 4; break;
    case ORC_SCALARS: src = h->scal; n = 8 * 8; break;
    case ORC_GFX: src = h->gfx; n = nu * 4; break;
    case ORC_GS: src = h->GS; n = C * 8; break;
    case ORC_NA: src = h->nA; n = C * 4; break;
    case ORC_RBA: src = h->RbA; n = C * 8; break;
    default: return -1;
    }
    if (bytes < n) return -2;
    memcpy(dst, src, n);
    return (int64_t)n;
}

/* ======================================================================================
 * Ego-motion compensation.  P:1550: "The vehicle speed and yaw rate are available
 * via CAN messages, so the ego movement of the test vehicle can be compensated in the grid map."  The
 * operation follows SPEC S:171-179 (ego_scroll): the grid content shifts by the integer-cell part of
 * (delta + residual) and the fraction is kept as the new residual; cells scrolled in at the leading edge
 * become vacuous (m_F = 0) and hold no particles; particles move by the same whole number of cells and
 * those that leave the grid become sentinel particles (A-19).  Readings (A-32): the integer
 * part is fp64 truncation toward zero of (delta + residual) / cell_size, the residual is
 * (delta + residual) - shift * cell_size in fp64; a particle moves by one f32 addition per coordinate;
 * a particle already at the sentinel position stays there; a shift of half the grid side or more is an
 * error and changes nothing.
 * ====================================================================================== */
int orc_ego_scroll(orc_ctx* h, double dx, double dy, int32_t* shift_x, int32_t* shift_y)
{
    const double cs = (double)h->p.cell_size;
    const double tx = dx + h->res_x, ty = dy + h->res_y;
    const double qx = trunc(tx / cs), qy = trunc(ty / cs);
    const int32_t W = h->p.width, H = h->p.height;
    if (!(fabs(qx) * 2.0 < (double)W) || !(fabs(qy) * 2.0 < (double)H)) return -1;
    const int32_t sx = (int32_t)qx, sy = (int32_t)qy;
    h->res_x = tx - qx * cs;
    h->res_y = ty - qy * cs;
    if (shift_x) *shift_x = sx;
    if (shift_y) *shift_y = sy;
    /* grid: the content of cell (r, c) moves to (r + sy, c + sx) */
    float* tmp = (float*)xcalloc(h->C, 4);
    for (int32_t r = 0; r < H; ++r)
        for (int32_t c = 0; c < W; ++c) {
            const int32_t r0 = r - sy, c0 = c - sx;
            tmp[(int64_t)r * W + c] = (r0 >= 0 && r0 < H && c0 >= 0 && c0 < W) ? h->m_free[(int64_t)r0 * W + c0] : 0.0f;
        }
    memcpy(h->m_free, tmp, h->C * 4);
    free(tmp);
    /* particles */
    for (int64_t i = 0; i < h->p.nu; ++i) {
        if (h->x[i] == SENTINEL_POS && h->y[i] == SENTINEL_POS) continue;
        const float xn = h->x[i] + (float)sx, yn = h->y[i] + (float)sy;
        if (xn >= 0.0f && xn < (float)W && yn >= 0.0f && yn < (float)H) {
            h->x[i] = xn; h->y[i] = yn;
        } else {
            h->x[i] = SENTINEL_POS; h->y[i] = SENTINEL_POS; h->vx[i] = 0.0f; h->vy[i] = 0.0f;
        }
    }
    return 0;
}

void orc_ego_residual(const orc_ctx* h, double* rx, double* ry)
{
    if (rx) *rx = h->res_x;
    if (ry) *ry = h->res_y;
}

/* ======================================================================================
 * Evaluation workload (PAPER section VIII, SPEC S:456-543 module "evaluation").
 * Mahalanobis distance (Eq. 88 `eq:mahadist`): m = v P^-1 v^T with P = [[var_x, cov_xy],
 * [cov_xy, var_y]] from Eqs. 81-84; written out for the 2x2 case in fp64:
 *   det = var_x var_y - cov_xy^2, m = (v_x^2 var_y - 2 v_x v_y cov_xy + v_y^2 var_x) / det.
 * Readings (A-33): P is regularised to P + 1e-6 I when det <= 1e-12; a cell
 * without reported moments has m = 0 (no velocity estimate: static); m is rounded once to f32.
 * Classification: dynamic detection iff m >= tau_m.  Cluster sums feed Eq. 85
 * `eq:mean_cluster` and Eq. 86 `eq:gaussian_mixture_x` on the host.
 * ====================================================================================== */
void orc_eval_cells(int64_t C, const float* mean, const float* cov, const uint8_t* valid, const uint8_t* labels,
                    const uint8_t* mask, const float* thr, int n_thr, float* m_out, uint64_t* counts, double* sums)
{
    if (counts) memset(counts, 0, sizeof(uint64_t) * 4 * (size_t)(n_thr > 0 ? n_thr : 0));
    if (sums) for (int i = 0; i < 5; ++i) sums[i] = 0.0;
    for (int64_t c = 0; c < C; ++c) {
        const double vx = mean[2 * c], vy = mean[2 * c + 1];
        double pxx = cov[3 * c], pyy = cov[3 * c + 1];
        const double pxy = cov[3 * c + 2];
        const int ok = valid ? valid[c] != 0 : (vx != 0.0 || vy != 0.0 || pxx != 0.0 || pyy != 0.0 || pxy != 0.0);
        double m = 0.0;
        if (ok) {
            double det = pxx * pyy - pxy * pxy;
            if (det <= 1e-12) {
                pxx = pxx + 1e-6;
                pyy = pyy + 1e-6;
                det = pxx * pyy - pxy * pxy;
            }
            const double num = (vx * vx * pyy - 2.0 * vx * vy * pxy) + vy * vy * pxx;
            m = num / det;
        }
        const float mf = (float)m;
        if (m_out) m_out[c] = mf;
        if (labels && counts && (labels[c] == 1 || labels[c] == 2)) {
            const int dyn = labels[c] == 2;
            for (int t = 0; t < n_thr; ++t) {
                const int det_dyn = mf >= thr[t];
                counts[4 * t + (dyn ? (det_dyn ? 0 : 1) : (det_dyn ? 2 : 3))] += 1;
            }
        }
        if (mask && sums && mask[c] && ok) {
            sums[0] += 1.0;
            sums[1] += vx;
            sums[2] += (double)cov[3 * c] + vx * vx;
            sums[3] += vy;
            sums[4] += (double)cov[3 * c + 1] + vy * vy;
        }
    }
}
