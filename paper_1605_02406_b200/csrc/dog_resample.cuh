// dog_resample.cuh -- one fused pass over the joint particle set: velocity moments (Alg. 6,
// Eqs. 81-84), new-born particle initialisation (Alg. 5) and systematic resampling (Alg. 7,
// Eq. 57) to the next state.
//
// Resampling is member-driven: every member of the joint list (the cell-sorted persistent particles
// and the birth slots, cell-interleaved, A-25) knows its cumulative fixed-point weight range
// [Q, Q') from its cell's joint prefix P_c and the even split of the cell's mass (A-23), and writes
// its copies to the outputs i with Q <= t_i < Q', t_i = floor((i 2^32 + U) W / (nu 2^32)) (A-24):
// i in [F(Q), F(Q')) with F(X) = #{i : t_i < X} = clamp(ceil((X nu 2^32 - U W) / (W 2^32)), 0, nu).
// This selects exactly what the oracle's binary search over the particle-level CDF selects; F is
// evaluated with an fp64 estimate corrected by exact 128-bit products (no 128-bit division).
#pragma once
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {

constexpr int kMomRange = 256;   // sorted slots per warp in the persistent part
struct MomPartial { double s[5]; };

struct RsConst {
    uint64_t W;
    uint32_t U, nu;
    double nu_over_W;  // nu / W  (fp64)
    double U_frac;     // U 2^-32  (exact)
    u128 UW;           // U * W
};

__device__ __forceinline__ RsConst make_rsconst(const DevScalars* sc, uint32_t nu)
{
    RsConst r;
    r.W = sc->W;
    r.U = sc->U;
    r.nu = nu;
    r.nu_over_W = r.W ? (double)nu / (double)r.W : 0.0;
    r.U_frac = (double)r.U * 0x1p-32;
    r.UW = (u128)r.U * (u128)r.W;
    return r;
}

// F(X) = number of systematic targets t_i below X = clamp(ceil(y), 0, nu) with
// y = (X nu 2^32 - U W) / (W 2^32) = X nu / W - U 2^-32.  The fp64 estimate of y is within 2^-20
// of y (|y| < 2^31, relative error < 2^-51); when it is further than 2^-16 from an integer its
// ceiling is exact, otherwise the ceiling is settled with exact 128-bit products.
__device__ __forceinline__ uint32_t fcount(uint64_t X, const RsConst& r)
{
    const double y = __fma_rn((double)X, r.nu_over_W, -r.U_frac);
    if (y <= -0.5) return 0u;
    if (y >= (double)r.nu) return r.nu;
    const double cy = ceil(y);
    const double d = cy - y;                       // in [0, 1)
    if (d > 0x1p-16 && d < 1.0 - 0x1p-16) return (uint32_t)cy;
    // exact: smallest q >= 0 with q W 2^32 >= X nu 2^32 - U W
    const u128 num0 = ((u128)X * (u128)r.nu) << 32;
    if (num0 <= r.UW) return 0u;
    const u128 num = num0 - r.UW;
    const u128 E = ((u128)r.W) << 32;
    uint64_t q = (uint64_t)fmax(cy - 1.0, 0.0);
    while ((u128)q * E < num) ++q;
    while (q > 0 && (u128)(q - 1) * E >= num) --q;
    return (uint32_t)(q < r.nu ? q : r.nu);
}

// Moments of cell c from its velocity sums (Eqs. 81-84 with the uniform weight w' = rho_p / S w_pred).
__device__ __forceinline__ void finalize_cell(uint32_t c, const double* s, uint32_t n, float rp, float w_pred,
                                              float2* __restrict__ mean, float* __restrict__ cov)
{
    const float S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));
    if (!(rp > 0.0f) || !(S > 0.0f)) return;
    const float w = __fmul_rn(__fdiv_rn(rp, S), w_pred);       // Eq. 71 with p_A = 0, Eq. 73
    const double wd = (double)w, rd = (double)rp;
    const double mx = wd * s[0] / rd, my = wd * s[1] / rd;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(wd * s[2] / rd - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(wd * s[3] / rd - my * my);
    cov[3 * (size_t)c + 2] = (float)(wd * s[4] / rd - mx * my);
}

struct NextState { float *x, *y, *vx, *vy; uint32_t* jidx; };
struct Pred { const float *x, *y, *vx, *vy; };
struct BirthDebug { float *x, *y, *vx, *vy; };
struct MomScratch { MomPartial* head; MomPartial* tail; uint32_t* tail_cell; uint8_t* head_ends; };

__global__ __launch_bounds__(256) void k_resample(
    const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ perm, Pred pr, CellList L, BlockTotals bt,
    uint32_t nblk, uint32_t chunk, const uint32_t* __restrict__ cell2list, NextState out, BirthDebug bdbg,
    float2* __restrict__ mean, float* __restrict__ cov, MomScratch ms, const DevScalars* __restrict__ sc,
    FilterConst fc, int64_t k, uint32_t pers_blocks, uint32_t nranges)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const RsConst rc = make_rsconst(sc, fc.nu);
    if (rc.W == 0) {   // empty world (A-26): every next particle goes to the sentinel
        for (uint32_t i = blockIdx.x * blockDim.x + tid; i < fc.nu; i += gridDim.x * blockDim.x) {
            out.x[i] = kSentinelPos; out.y[i] = kSentinelPos; out.vx[i] = 0.0f; out.vy[i] = 0.0f;
            if (out.jidx) out.jidx[i] = 0xFFFFFFFFu;
        }
    }

    if (blockIdx.x >= pers_blocks) {
        // ---------------- birth slots (Alg. 5): state from the slot's Philox draw, then copies
        const uint32_t s = (blockIdx.x - pers_blocks) * blockDim.x + tid;
        if ((uint64_t)s >= sc->s_total) return;
        uint32_t blo = 0, bhi = nblk;              // last cell chunk with first slot <= s
        while (bhi - blo > 1) {
            const uint32_t mid = (blo + bhi) >> 1;
            if (bt.s0[mid] <= s) blo = mid; else bhi = mid;
        }
        uint32_t lo = blo * chunk, hi = lo + bt.cnt[blo];   // last entry of the chunk with sb <= s
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (L.sb[mid] <= s) lo = mid; else hi = mid;
        }
        const uint32_t li = lo;
        const uint32_t r = s - L.sb[li];
        const uint32_t c = L.c[li];
        const uint32_t col = c % (uint32_t)fc.W, row = c / (uint32_t)fc.W;
        const Philox4 d = draw(fc.seed, s, k, STAGE_BIRTH);
        const float colf = (float)col, rowf = (float)row;
        float bx = __fadd_rn(colf, unit24(d.r0));
        float by = __fadd_rn(rowf, unit24(d.r1));
        const float cx1 = __fadd_rn(colf, 1.0f), cy1 = __fadd_rn(rowf, 1.0f);
        if (bx >= cx1) bx = __int_as_float(__float_as_int(cx1) - 1);    // nextafter(col+1, 0) (A-16)
        if (by >= cy1) by = __int_as_float(__float_as_int(cy1) - 1);
        float n0, n1;
        box_muller(d.r2, d.r3, n0, n1);
        float bvx = __fmul_rn(fc.sigma_b, n0), bvy = __fmul_rn(fc.sigma_b, n1);
        if (fc.v_max > 0.0f) {
            bvx = fminf(fmaxf(bvx, -fc.v_max), fc.v_max);
            bvy = fminf(fmaxf(bvy, -fc.v_max), fc.v_max);
        }
        if (bdbg.x) { bdbg.x[s] = bx; bdbg.y[s] = by; bdbg.vx[s] = bvx; bdbg.vy[s] = bvy; }
        if (rc.W == 0) return;
        const uint64_t bb = L.bb[li];
        const uint32_t rbm = L.rb[li];
        const uint64_t Q0 = bt.P0[li / chunk] + L.Pl[li] + L.Rp[li] + (uint64_t)r * bb + min(r, rbm);
        const uint64_t Q1 = Q0 + bb + (r < rbm ? 1u : 0u);
        const uint32_t o0 = fcount(Q0, rc), o1 = fcount(Q1, rc);
        const uint32_t joint = L.start[li] + L.sb[li] + L.n[li] + r;
        for (uint32_t o = o0; o < o1; ++o) {
            out.x[o] = bx; out.y[o] = by; out.vx[o] = bvx; out.vy[o] = bvy;
            if (out.jidx) out.jidx[o] = joint;
        }
        return;
    }

    // ---------------- persistent members: one warp per range of 256 cell-sorted slots
    const uint32_t wr = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    if (wr >= nranges) return;
    const uint32_t n_in = (uint32_t)sc->n_in;
    const float w_pred = sc->w_pred;
    const uint32_t start = wr * kMomRange;
    if (start >= n_in) {
        if (lane == 0) { ms.tail_cell[wr] = 0xFFFFFFFFu; ms.head_ends[wr] = 1; }
        return;
    }
    const uint32_t end = min(start + (uint32_t)kMomRange, n_in);
    const uint32_t first_cell = skeys[start];
    const bool cont_before = start > 0 && skeys[start - 1] == first_cell;
    bool have_carry = false;
    uint32_t carry_cell = 0xFFFFFFFFu;
    double carry[5] = {0, 0, 0, 0, 0};

    for (uint32_t j0 = start; j0 < end; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool valid = j < end;
        const uint32_t cell = valid ? skeys[j] : 0xFFFFFFFEu;
        const uint32_t cell_next = (j + 1 < n_in) ? skeys[j + 1] : 0xFFFFFFFFu;
        uint32_t li = 0, cst = 0, cn = 0;
        float crho = 0.0f;
        double v[5] = {0, 0, 0, 0, 0};
        if (valid) {
            li = cell2list[cell];
            cst = L.start[li];
            cn = L.n[li];
            crho = L.rho_p[li];
            const uint32_t src = perm[j];
            const float X = pr.x[src], Y = pr.y[src], VX = pr.vx[src], VY = pr.vy[src];
            const double a = (double)VX, bq = (double)VY;
            v[0] = a; v[1] = bq; v[2] = a * a; v[3] = bq * bq; v[4] = a * bq;
            if (rc.W) {
                const uint32_t r = j - cst;
                const uint64_t bp = L.bp[li];
                const uint32_t rpm = L.rp[li];
                const uint64_t Q0 = bt.P0[li / chunk] + L.Pl[li] + (uint64_t)r * bp + min(r, rpm);
                const uint64_t Q1 = Q0 + bp + (r < rpm ? 1u : 0u);
                const uint32_t o0 = fcount(Q0, rc), o1 = fcount(Q1, rc);
                const uint32_t joint = cst + L.sb[li] + r;
                for (uint32_t o = o0; o < o1; ++o) {
                    out.x[o] = X; out.y[o] = Y; out.vx[o] = VX; out.vy[o] = VY;
                    if (out.jidx) out.jidx[o] = joint;
                }
            }
        }
        // segmented inclusive scan of the velocity sums within the 32-slot chunk
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t oc = __shfl_up_sync(0xffffffffu, cell, off);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const double o = __shfl_up_sync(0xffffffffu, v[q], off);
                if (lane >= off && oc == cell) v[q] += o;
            }
        }
        if (have_carry && cell == carry_cell) {
#pragma unroll
            for (int q = 0; q < 5; ++q) v[q] += carry[q];
        }
        const bool seg_end = valid && cell_next != cell;
        if (seg_end) {
            if (cell == first_cell && cont_before) {
                MomPartial hp;
#pragma unroll
                for (int q = 0; q < 5; ++q) hp.s[q] = v[q];
                ms.head[wr] = hp;
                ms.head_ends[wr] = 1;
            } else {
                finalize_cell(cell, v, cn, crho, w_pred, mean, cov);
            }
        }
        const int last = (int)min(31u, end - 1 - j0);
        const uint32_t lc = __shfl_sync(0xffffffffu, cell, last);
        const bool lend = __shfl_sync(0xffffffffu, (int)seg_end, last) != 0;
#pragma unroll
        for (int q = 0; q < 5; ++q) carry[q] = __shfl_sync(0xffffffffu, v[q], last);
        have_carry = !lend;
        carry_cell = lc;
    }
    if (lane == 0) {
        if (have_carry) {
            MomPartial p;
#pragma unroll
            for (int q = 0; q < 5; ++q) p.s[q] = carry[q];
            if (carry_cell == first_cell && cont_before) {   // the range lies inside one segment
                ms.head[wr] = p;
                ms.head_ends[wr] = 0;
                ms.tail_cell[wr] = 0xFFFFFFFFu;
            } else {
                ms.tail[wr] = p;
                ms.tail_cell[wr] = carry_cell;
                if (!cont_before) ms.head_ends[wr] = 1;
            }
        } else {
            ms.tail_cell[wr] = 0xFFFFFFFFu;
            if (!cont_before) ms.head_ends[wr] = 1;
        }
    }
}

// Segments spanning several warp ranges: tail partial of the range where the segment starts plus the
// head partials of the following ranges, in a fixed order (deterministic).
__global__ void k_moments_fixup(MomScratch ms, CellList L, const uint32_t* __restrict__ cell2list,
                                float2* __restrict__ mean, float* __restrict__ cov,
                                const DevScalars* __restrict__ sc, uint32_t nranges)
{
    const uint32_t wr = blockIdx.x * blockDim.x + threadIdx.x;
    if (wr >= nranges) return;
    const uint32_t c = ms.tail_cell[wr];
    if (c == 0xFFFFFFFFu) return;
    double s[5];
    for (int q = 0; q < 5; ++q) s[q] = ms.tail[wr].s[q];
    for (uint32_t r = wr + 1; r < nranges; ++r) {
        for (int q = 0; q < 5; ++q) s[q] += ms.head[r].s[q];
        if (ms.head_ends[r]) break;
    }
    const uint32_t li = cell2list[c];
    finalize_cell(c, s, L.n[li], L.rho_p[li], sc->w_pred, mean, cov);
}

}  // namespace dog
