// dog_cells.cuh -- per-cell stages of the cycle (Alg. 3, Alg. 5 slot allocation, Alg. 7 joint CDF).
//
// k_cells: one pass over the grid.  For every cell: n_c (from k_predict_sort's counts), S_c = n_c w_pred
// (Eq. 61, exact), m_p = min(S_c, occ_max) (Eq. 17), m_Fp = min(alpha m_F, 1 - m_p) (Eq. 62),
// Dempster update (Eq. 63), birth split (Eqs. 67-68), fixed-point masses (A-23) and the readouts.
// Cells holding particles or receiving born mass ("active" cells, typically ~1 % of the grid) are
// staged, in cell order, in their block's segment of a staging list (each block owns a contiguous chunk
// of cells, so no grid-wide scan is needed); the last block to finish turns the per-block counts into
// offsets, so (block, position) maps to a position in one flat, cell-ordered active list.
//
// k_list_scan (persistent blocks over 2048-entry tiles of the flat active list, decoupled look-back):
// gathers the staged entries into the flat list, first sorted slot of each cell (prefix of n_c),
// born-mass CDF A_c (prefix of R_b) -> exact slot allocation s_c = floor((2 nu_b A_c + A) / (2A))
// (A-15), the gated joint mass J_c = R_p + [n_b > 0] R_b and its prefix (the joint CDF in
// cell-interleaved order, A-25), the even-split parameters, the birth work items (<= 256 slots of one
// cell) and the run-list offsets.  The tile holding the last entry publishes W, w_bar (Eq. 57), U (A-24).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {

#ifndef BIRTH_ITEM
#define BIRTH_ITEM 256
#endif
constexpr uint32_t kItem = BIRTH_ITEM;   // birth slots per k_births work item

struct StageList {          // k_cells staging, capacity nblk * chunk (>= C); entry li belongs to block li / chunk
    uint32_t* c;            // cell index
    uint32_t* n;            // persistent particles n_c
    uint64_t* Rp;           // floor(rho_p 2^FX) (0 if n_c = 0)
    uint64_t* Rb;           // floor(rho_b 2^FX) if m_zO > 0 else 0
    float* rho_p;           // f32 rho_p (moments denominator)
    uint32_t* np;           // runs ("pairs") of the cell over the sort tiles
};

struct BirthRec {           // what the birth kernels need of an entry with birth slots: one 32-byte load
    uint64_t PB;            // P_c + R_p: joint-CDF position of the cell's first birth (this context)
    uint64_t bb;            // R_b / n_b
    uint32_t c, nb, sb, rb; // cell, birth slots, first slot (global), R_b mod n_b
};

struct CellList {           // the flat active list in cell order (SoA, capacity C)   (k_list_scan)
    uint32_t* c;            // cell index
    uint32_t* n;            // persistent particles n_c
    uint64_t* Rp;           // floor(rho_p 2^FX)
    float* rho_p;           // f32 rho_p
    uint32_t* start;        // first cell-sorted slot of the cell
    uint32_t* sb;           // first birth slot of the cell (global)
    uint32_t* nb;           // birth slots of the cell
    uint64_t* P;            // exclusive joint-CDF prefix (A-25)
    uint32_t* it;           // exclusive birth work-item prefix
    uint64_t* bp;           // R_p / n_c        (even split of R_p)
    uint32_t* rp;           // R_p mod n_c
    uint64_t* bb;           // R_b / n_b
    uint32_t* rb;           // R_b mod n_b
    uint32_t* np;           // runs of the cell
    uint32_t* ps;           // exclusive prefix of np (offset of the cell's run list)
    uint32_t* pfill;        // run-list fill counter (reset here, k_pair_fill)
    BirthRec* brec;         // entries with n_b > 0 only (written with P; the others hold stale records)
};

struct BlockTotals {        // one entry per cell chunk (k_cells); prefixes / totals are formed in k_list_scan
    uint32_t* cnt;          // active cells staged by the block
    uint64_t* n0;           // sum of n_c over them
    uint64_t* rb0;          // sum of R_b over them
    uint32_t* np0;          // sum of their run counts
};

// floor(max(m, 0) 2^FX) (A-23): exact (a power-of-two scale)
__device__ __forceinline__ uint64_t fxq(float m, const FilterConst& fc)
{
    return (m > 0.0f) ? __double2ull_rz(__dmul_rn((double)m, fc.fx)) : 0ull;
}

// e^q for q <= 0 (A-34 "exp spec")
__device__ __forceinline__ float exp_spec(float q)
{
    if (!(q >= -87.0f)) return 0.0f;
    if (q > 0.0f) q = 0.0f;
    const float kf = rintf(__fmul_rn(q, 1.44269504088896341f));
    float r = __fmaf_rn(-kf, 0.693359375f, q);
    r = __fmaf_rn(-kf, -2.12194440e-4f, r);
    const float z = __fmul_rn(r, r);
    float y = 1.9875691500e-4f;
    y = __fmaf_rn(y, r, 1.3981999507e-3f);
    y = __fmaf_rn(y, r, 8.3334519073e-3f);
    y = __fmaf_rn(y, r, 4.1665795894e-2f);
    y = __fmaf_rn(y, r, 1.6666665459e-1f);
    y = __fmaf_rn(y, r, 5.0000001201e-1f);
    y = __fmaf_rn(y, z, r);
    y = __fadd_rn(y, 1.0f);
    const int k = (int)kf;                                   // -126 <= k <= 0
    return __fmul_rn(y, __int_as_float((127 + k) << 23));
}

struct CellOut {
    uint32_t n;
    float S, mO, mF, rp, rb;
    uint64_t Rp, Rb;
    bool bad;
};

// Alg. 3 for one cell, canonical operation order of DESIGN.md 3.2 (bit-identical to the oracle).
// Divisions by exactly 1 and of exactly 0 are skipped: IEEE gives the same result without them.
__device__ __forceinline__ CellOut cell_math(uint32_t n, float m_free, float2 z, float w_pred, float alpha,
                                             const FilterConst& fc)
{
    CellOut o;
    o.n = n;
    if (n == 0 && z.x == 0.0f && z.y == 0.0f && __float_as_uint(z.x) == 0u) {
        // empty cell under a vacuous measurement: the general path below yields exactly these values
        // (S = +0, K = 0, 1-K = 1, m_O = +0, m_F = m_Fp, rho_b = rho_p = +0, R = 0)
        o.S = 0.0f; o.mO = 0.0f; o.rp = 0.0f; o.rb = 0.0f; o.Rp = 0ull; o.Rb = 0ull; o.bad = false;
        o.mF = fminf(__fmul_rn(alpha, m_free), 1.0f);
        return o;
    }
    o.S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));        // Eq. 61, exact
    const float m_p = fminf(o.S, fc.occ_max);                              // Eq. 17 cap (A-7)
    const float m_fp = fminf(__fmul_rn(alpha, m_free), __fsub_rn(1.0f, m_p));   // Eq. 62
    o.bad = !(z.x >= 0.0f) || !(z.y >= 0.0f) || !(__fadd_rn(z.x, z.y) <= kMeasSumMax);
    if (o.bad) z = make_float2(0.0f, 0.0f);                                // A-27
    const float aO = m_p, aF = m_fp, aW = __fsub_rn(__fsub_rn(1.0f, aO), aF);
    const float bO = z.x, bF = z.y, bW = __fsub_rn(__fsub_rn(1.0f, bO), bF);
    const float K = __fadd_rn(__fmul_rn(aO, bF), __fmul_rn(aF, bO));
    const float oneK = __fsub_rn(1.0f, K);
    if (oneK <= 0.0f) { o.mO = bO; o.mF = bF; }                            // A-10
    else {
        const float nO = __fadd_rn(__fmul_rn(aO, bO), __fadd_rn(__fmul_rn(aO, bW), __fmul_rn(aW, bO)));
        const float nF = __fadd_rn(__fmul_rn(aF, bF), __fadd_rn(__fmul_rn(aF, bW), __fmul_rn(aW, bF)));
        if (oneK == 1.0f) { o.mO = nO; o.mF = nF; }
        else { o.mO = __fdiv_rn(nO, oneK); o.mF = __fdiv_rn(nF, oneK); }
    }
    const float q = __fmul_rn(fc.p_b, __fsub_rn(1.0f, m_p));               // Eqs. 67-68 (A-11)
    const float den = __fadd_rn(m_p, q);
    const float mq = __fmul_rn(o.mO, q);
    o.rb = den > 0.0f ? (mq == 0.0f ? mq : __fdiv_rn(mq, den)) : 0.0f;     // (+-0)/den = +-0
    o.rp = __fsub_rn(o.mO, o.rb);
    o.Rp = n > 0 ? fxq(o.rp, fc) : 0ull;                                      // A-23
    o.Rb = z.x > 0.0f ? fxq(o.rb, fc) : 0ull;                                 // P:1197 gate (A-13)
    return o;
}

// The exact PHD/MIB cell update (NEXT-3, A-37; Eqs. 31-32, 38-42 with a uniform likelihood equal to
// the clutter density, the section IV-F setting): obs = (occurred, p_TP, p_FP, -).  f32 in the order of
// orc_exact_cell.  occupancy = rho_p + rho_b (mO), free = 1 - occupancy (mF); births wherever r_b > 0.
__device__ __forceinline__ CellOut cell_math_exact(uint32_t n, float4 obs, float w_pred, const FilterConst& fc)
{
    CellOut o;
    o.n = n;
    o.S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));        // Eq. 31, exact
    const float rpp = fminf(o.S, fc.occ_max);                              // truncation
    const float rbp = __fmul_rn(fc.p_b, __fsub_rn(1.0f, rpp));             // Eq. 32
    const float rplus = __fadd_rn(rpp, rbp), rbar = __fsub_rn(1.0f, rplus);
    float num, den;
    if (obs.x > 0.0f) {                                                    // Eqs. 38-40 (g_A = p_cl cancels)
        num = obs.y;
        den = __fadd_rn(__fmul_rn(obs.z, rbar), __fmul_rn(obs.y, rplus));
    } else {                                                               // Eq. 41
        num = __fsub_rn(1.0f, obs.y);
        den = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, obs.z), rbar), __fmul_rn(num, rplus));
    }
    const float f = den > 0.0f ? __fdiv_rn(num, den) : 0.0f;
    o.rp = __fmul_rn(rpp, f);
    o.rb = __fmul_rn(rbp, f);
    o.mO = __fadd_rn(o.rp, o.rb);                                          // Eq. 42
    o.mF = __fsub_rn(1.0f, o.mO);
    o.Rp = n > 0 ? fxq(o.rp, fc) : 0ull;
    o.Rb = fxq(o.rb, fc);
    o.bad = false;
    return o;
}

// The exact filter with a single-object likelihood (NEXT-3 general form, A-38): cells where
// a measurement occurred and p_A > 0 take the g_A update of cell_math_exact_lik.  pA == nullptr: off.
struct ExactLik {
    const float* pA;          // [C] association probability
    const float4* lik;        // [C] (u_x, u_y, v_r, sd)
    uint64_t* GSc;            // [C] sum of the members' gfx (k_dopp_runs); cleared here after reading
    const uint32_t* gmax;     // [C] largest member likelihood (f32 bits, A-34)
    float* pAe;               // [C] out: effective association weight of the members' split
    float* pic;               // [C] out: associated share of the births
};

__device__ __forceinline__ bool lik_cell(const ExactLik& xl, float4 ob, uint32_t c)
{
    return xl.pA && ob.x > 0.0f && xl.pA[c] > 0.0f;
}

// E[g] of a new-born object under the birth prior v ~ N(0, sigma_B^2 I): N(v_r; 0, sd^2 + sigma_B^2)
// (A-38), f32 in the order of the oracle's orc_birth_mean_lik
__device__ __forceinline__ float birth_mean_lik(float vr, float sd, float sigma_b)
{
    const float s = __fsqrt_rn(__fadd_rn(__fmul_rn(sd, sd), __fmul_rn(sigma_b, sigma_b)));
    const float t = __fdiv_rn(vr, s);
    const float q = __fmul_rn(__fmul_rn(t, t), -0.5f);
    return __fdiv_rn(exp_spec(q), __fmul_rn(s, 2.50662827463100050f));
}

// Eqs. 49-52 with g_A = p_A g + (1 - p_A) p_cl for a cell with a measurement (A-38): the fp64 sums in
// the oracle's written order (orc_exact_lik_cell), r_p+, r_b+ as cell_math_exact.  pAe / pi returned.
__device__ __forceinline__ CellOut cell_math_exact_lik(uint32_t n, float4 ob, float w_pred, const FilterConst& fc,
                                                       float pA, float4 d, uint64_t GS, float gmax, float& pAe,
                                                       float& pi)
{
    CellOut o;
    o.n = n;
    o.S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));
    const float rpp = fminf(o.S, fc.occ_max);
    const float rbp = __fmul_rn(fc.p_b, __fsub_rn(1.0f, rpp));
    const float rplus = __fadd_rn(rpp, rbp), rbar = __fsub_rn(1.0f, rplus);
    const double pa = (double)pA, cl = (double)ob.w;
    const double Sg = __dmul_rn(__dmul_rn(__ull2double_rn(GS), 0x1p-31), (double)gmax);
    const double gA_sum = __dadd_rn(__dmul_rn(pa, Sg), __dmul_rn(__dmul_rn((double)n, __dsub_rn(1.0, pa)), cl));
    const double gp = n ? __ddiv_rn(gA_sum, (double)n) : 0.0;
    const double Eb = (double)birth_mean_lik(d.z, d.w, fc.sigma_b);
    const double gb = __dadd_rn(__dmul_rn(pa, Eb), __dmul_rn(__dsub_rn(1.0, pa), cl));
    const double num_p = __dmul_rn(__dmul_rn((double)ob.y, (double)rpp), gp);
    const double num_b = __dmul_rn(__dmul_rn((double)ob.y, (double)rbp), gb);
    const double mu = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn((double)ob.z, cl), (double)rbar), num_p), num_b);
    o.rp = mu > 0.0 ? __double2float_rn(__ddiv_rn(num_p, mu)) : 0.0f;
    o.rb = mu > 0.0 ? __double2float_rn(__ddiv_rn(num_b, mu)) : 0.0f;
    pAe = gA_sum > 0.0 ? __double2float_rn(__ddiv_rn(__dmul_rn(pa, Sg), gA_sum)) : 0.0f;
    pi = gb > 0.0 ? __double2float_rn(__ddiv_rn(__dmul_rn(pa, Eb), gb)) : 0.0f;
    o.mO = __fadd_rn(o.rp, o.rb);
    o.mF = __fsub_rn(1.0f, o.mO);
    o.Rp = n > 0 ? fxq(o.rp, fc) : 0ull;
    o.Rb = fxq(o.rb, fc);
    o.bad = false;
    return o;
}

// the exact update of cell c: with the likelihood where lik_cell, else cell_math_exact.  commit: the
// final evaluation of an active cell -- writes pAe / pi and clears the cell's GS accumulator.
__device__ __forceinline__ CellOut cell_exact_any(uint32_t n, float4 ob, uint32_t c, float w_pred, const FilterConst& fc,
                                                  const ExactLik& xl, bool commit)
{
    if (!lik_cell(xl, ob, c)) return cell_math_exact(n, ob, w_pred, fc);
    const uint64_t GS = xl.GSc[c];
    float pAe, pi;
    const CellOut o = cell_math_exact_lik(n, ob, w_pred, fc, xl.pA[c], xl.lik[c], GS, __uint_as_float(xl.gmax[c]), pAe, pi);
    if (commit) {
        xl.pAe[c] = pAe;
        xl.pic[c] = pi;
        if (GS) xl.GSc[c] = 0ull;
    }
    return o;
}

constexpr int kCellThreads = 256, kCellItems = 8, kCellIter = kCellThreads * kCellItems;   // 2048 cells
constexpr int kMaxCellBlocks = 4096;

struct CellDebug { float* rho_p; float* rho_b; uint64_t* Rp; uint64_t* Rb; };

// Exclusive prefix of v[0..m) in place (one block, 256 threads), returns the total.
template <typename T>
__device__ __forceinline__ T block_prefix_inplace(T* v, uint32_t m, T* s_scan)
{
    T carry = 0;
    for (uint32_t b0 = 0; b0 < m; b0 += blockDim.x * 8) {
        T x[8], sum = 0;
        const uint32_t b = b0 + threadIdx.x * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) { x[i] = b + i < m ? __ldcg(v + b + i) : T(0); sum += x[i]; }
        T tot;
        T run = carry + block_excl_scan<T, 8>(sum, s_scan, tot);
#pragma unroll
        for (int i = 0; i < 8; ++i) { if (b + i < m) v[b + i] = run; run += x[i]; }
        carry += tot;
    }
    return carry;
}

// Block b owns cells [b chunk, (b+1) chunk), 2048 per iteration; item i of thread t in an iteration
// is cell base + i*256 + t (coalesced; one warp = one 32-bit word of the moments-valid bitmask).  All
// loads of an iteration are issued up front.  Active cells (~1 %) keep their inputs (n_c, m_F) untouched
// in the first pass; after the block's staging offsets are known they are recomputed from them
// (identical arithmetic) and staged, and only then is m_F updated and n_c cleared.
// kExact: the exact PHD/MIB update from obs[C] (NEXT-3) instead of Dempster's rule from meas; m_F untouched.
template <bool kExact>
#ifndef CELL_MINB
#define CELL_MINB 4
#endif
__global__ __launch_bounds__(kCellThreads, CELL_MINB) void k_cells(
    uint32_t* __restrict__ counts, uint32_t* __restrict__ npairs, float* __restrict__ m_free, const float2* __restrict__ meas,
    float* __restrict__ occ, float* __restrict__ free_out, float2* __restrict__ mean, float* __restrict__ cov,
    uint32_t* __restrict__ mvalid, CellDebug dbg, StageList L, BlockTotals bt, uint32_t chunk, DevScalars* sc, FilterConst fc, float alpha,
    const float4* __restrict__ obs, ExactLik xl, uint32_t dense)
{
    PDL_ENTER();
    __shared__ uint32_t s_cnt[kCellItems][kCellThreads / 32];
    __shared__ uint32_t s_run;
    __shared__ uint64_t s_A[9], s_N[9];
    __shared__ uint32_t s_bad[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const float w_pred = scrd(sc->w_pred);
    const uint32_t c0 = blockIdx.x * chunk;
    const uint32_t c1 = min(c0 + chunk, fc.C);
    const uint32_t lbase = blockIdx.x * chunk;
    if (tid == 0) s_run = 0;

    uint64_t A_loc = 0, N_loc = 0;
    uint32_t bad_loc = 0, P_loc = 0;
    for (uint32_t base = c0; base < c1; base += kCellIter) {
        uint32_t n[kCellItems], prev[kCellItems];
        float mf[kCellItems];
        float2 z[kCellItems];
        float4 ob[kCellItems];
        uint32_t npf[kCellItems];            // kExact: every cell is active -> run counts loaded up front
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            const uint32_t c = base + i * kCellThreads + tid;
            const bool valid = c < c1;
            n[i] = valid ? counts[c] : 0u;
            if (kExact) {
                ob[i] = valid ? obs[c] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                npf[i] = valid ? npairs[c] : 0u;
            } else {
                mf[i] = valid ? m_free[c] : 0.0f;
                z[i] = valid ? meas[c] : make_float2(0.0f, 0.0f);
            }
            const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
            prev[i] = (lane == 0 && (word << 5) < c1) ? mvalid[word] : 0u;
        }
        uint32_t abal[kCellItems];
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            const uint32_t c = base + i * kCellThreads + tid;
            const bool valid = c < c1;
            const bool inl = kExact && dense;                // dense exact cycles: the entry is written here
            const CellOut o = kExact ? cell_exact_any(n[i], ob[i], c, w_pred, fc, xl, inl && valid)
                                     : cell_math(n[i], mf[i], z[i], w_pred, alpha, fc);
            const bool vnow = valid && o.n > 0 && o.rp > 0.0f && o.S > 0.0f;
            const uint32_t bal = __ballot_sync(0xffffffffu, vnow);
            const uint32_t pw = __shfl_sync(0xffffffffu, prev[i], 0);
            const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
            const bool act = valid && (dense || o.n > 0 || o.Rb > 0);   // dense: every cell is an entry (li = c)
            if (valid) {
                occ[c] = o.mO;
                free_out[c] = o.mF;
                if (!kExact && !act) m_free[c] = o.mF;  // Alg. 3 store_values (active cells: below)
                if (!vnow && ((pw >> lane) & 1u)) {     // moments were reported last cycle: clear (A-18)
                    mean[c] = make_float2(0.0f, 0.0f);
                    cov[3 * (size_t)c] = 0.0f; cov[3 * (size_t)c + 1] = 0.0f; cov[3 * (size_t)c + 2] = 0.0f;
                }
                if (dbg.rho_p) {
                    dbg.rho_p[c] = o.rp; dbg.rho_b[c] = o.rb; dbg.Rp[c] = o.Rp; dbg.Rb[c] = o.Rb;
                }
                bad_loc += o.bad ? 1u : 0u;
            }
            if (lane == 0 && (word << 5) < c1 && bal != pw) mvalid[word] = bal;
            if (inl) {                                      // entry li = c (the list is the grid, no staging)
                if (valid) {
                    if (o.n) counts[c] = 0u;
                    L.c[c] = c; L.n[c] = o.n; L.Rp[c] = o.Rp; L.Rb[c] = o.Rb; L.rho_p[c] = o.rp;
                    uint32_t npc = 0;
                    if (o.n) { npc = npf[i]; npairs[c] = 0u; }
                    L.np[c] = npc;
                    A_loc += o.Rb;
                    N_loc += o.n;
                    P_loc += npc;
                }
                continue;
            }
            abal[i] = __ballot_sync(0xffffffffu, act);
            if (lane == 0) s_cnt[i][warp] = __popc(abal[i]);
        }
        if (kExact && dense) {                              // block-uniform
            if (tid == 0) s_run += min(c1 - base, (uint32_t)kCellIter);
            __syncthreads();
            continue;
        }
        __syncthreads();
        if (warp == 0) {   // exclusive offsets in cell order (item-major, then warp) + running total
            const uint32_t v0 = s_cnt[lane >> 3][lane & 7], v1 = s_cnt[4 + (lane >> 3)][lane & 7];
            const uint32_t i0 = warp_incl_scan(v0, lane), i1 = warp_incl_scan(v1, lane);
            const uint32_t t0 = __shfl_sync(0xffffffffu, i0, 31);
            const uint32_t run = s_run;
            s_cnt[lane >> 3][lane & 7] = run + i0 - v0;
            s_cnt[4 + (lane >> 3)][lane & 7] = run + t0 + i1 - v1;
            __syncwarp();
            if (lane == 31) s_run = run + t0 + i1;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            if ((abal[i] >> lane) & 1u) {               // active cell: same inputs (untouched), same arithmetic
                const uint32_t c = base + i * kCellThreads + tid;
                // exact filter: the inputs are still in registers (no reload: every cell comes here)
                const CellOut o = kExact ? cell_exact_any(n[i], ob[i], c, w_pred, fc, xl, true)
                                         : cell_math(__ldcg(counts + c), __ldcg(m_free + c), meas[c], w_pred, alpha, fc);
                if (!kExact) m_free[c] = o.mF;
                if (o.n) counts[c] = 0u;                // ready for the next cycle's k_predict_sort
                const uint32_t li = lbase + s_cnt[i][warp] + __popc(abal[i] & lt);
                DOG_ASSERT(li < lbase + chunk);
                L.c[li] = c; L.n[li] = o.n; L.Rp[li] = o.Rp; L.Rb[li] = o.Rb; L.rho_p[li] = o.rp;
                uint32_t npc = 0;
                if (o.n) { npc = kExact ? npf[i] : npairs[c]; npairs[c] = 0u; }
                L.np[li] = npc;
                A_loc += o.Rb;
                N_loc += o.n;
                P_loc += npc;                               // (the grid-wide list scan's chunk totals)
            }
        }
        __syncthreads();
    }
    // block totals (integers: order-independent)
    A_loc = warp_sum(A_loc);
    N_loc = warp_sum(N_loc);
    P_loc = warp_sum(P_loc);
    bad_loc = warp_sum(bad_loc);
    __shared__ uint32_t s_P[8];
    if (lane == 0) { s_A[warp] = A_loc; s_N[warp] = N_loc; s_bad[warp] = bad_loc; s_P[warp] = P_loc; }
    __syncthreads();
    if (tid == 0) {
        uint64_t A = 0, N = 0; uint32_t b = 0;
        uint32_t np = 0;
        for (int w = 0; w < kCellThreads / 32; ++w) { A += s_A[w]; N += s_N[w]; b += s_bad[w]; np += s_P[w]; }
        bt.cnt[blockIdx.x] = s_run;
        bt.np0[blockIdx.x] = np;
        bt.n0[blockIdx.x] = N;
        bt.rb0[blockIdx.x] = A;
        if (b) atomicAdd(&sc->meas_bad, b);
        if (A) atomicAdd((unsigned long long*)&sc->A_acc, (unsigned long long)A);   // integer: order-free
    }
}

// ------------------------------------------------------------------------------------------------
// exact floor((2 nu_b X + A) / (2A)) for X <= A < 2^64 without a 128-bit division: fp64 estimate
// (rcpA = 1/A rounded, shared by all cells), then exact integer correction (the quotient is
// <= nu_b < 2^30; the estimate is within one of it).
__device__ __forceinline__ uint64_t slot_of(uint64_t X, uint64_t A, uint64_t nu_b, double rcpA)
{
    if (A == 0) return 0;
    const u128 num = (u128)2 * (u128)nu_b * (u128)X + (u128)A;
    const u128 den = (u128)2 * (u128)A;
    uint64_t q = (uint64_t)floor(fma((double)X * rcpA, (double)nu_b, 0.5));
    while (q > 0 && (u128)q * den > num) --q;
    while ((u128)(q + 1) * den <= num) ++q;
    return q;
}
__device__ __forceinline__ uint64_t slot_of(uint64_t X, uint64_t A, uint64_t nu_b)
{
    return slot_of(X, A, nu_b, A ? 1.0 / (double)A : 0.0);
}

// floor(a / d) and a mod d for a < 2^53, 0 < d < 2^32 (fixed-point masses are <= 2^40): the fp64
// estimate a * (1/d) is within one of the exact quotient; one integer correction settles it.
__device__ __forceinline__ uint64_t divmod53(uint64_t a, uint32_t d, uint32_t& r)
{
    const double est = __dmul_rn((double)a, __drcp_rn((double)d));
    uint64_t q = est > 0.0 ? (uint64_t)est : 0ull;
    int64_t rem = (int64_t)(a - q * (uint64_t)d);
    if (rem < 0) { --q; rem += d; }
    else if (rem >= (int64_t)d) { ++q; rem -= d; }
    r = (uint32_t)rem;
    return q;
}

// k_list_scan runs as ONE thread-block cluster (kLsCluster CTAs of 1024 threads on as many SMs): the two
// dependent prefix sums over the active list -- (n_c, runs, R_b) and then (J_c, birth work items) --
// are exchanged between the CTAs through distributed shared memory with cluster barriers, so no
// global-memory look-back chain is needed.  The list is processed in rounds of kLsCluster*1024*kLsItems
// entries (one round for typical scenes).
constexpr int kLsThreads = 1024, kLsWarps = kLsThreads / 32, kLsItems = 2;
constexpr int kLsClusterMax = 16;

// Exclusive prefix over a warp's 32*I entries laid out entry = i*32 + lane (so loads and stores of
// consecutive entries coalesce); returns the warp total.
template <int I>
__device__ __forceinline__ uint64_t warp_excl_items(const uint64_t (&v)[I], uint64_t (&ex)[I])
{
    const int lane = threadIdx.x & 31;
    uint64_t carry = 0;
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const uint64_t inc = warp_incl_scan(v[i], lane);
        ex[i] = carry + inc - v[i];
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    return carry;
}

// Block-level exclusive scan of one ulonglong2 per thread (this CTA only); returns the CTA total.
__device__ __forceinline__ ulonglong2 cta_excl_scan2(ulonglong2 v, ulonglong2* s_w, ulonglong2& off)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t ix = warp_incl_scan(v.x, lane), iy = warp_incl_scan(v.y, lane);
    if (lane == 31) s_w[warp] = make_ulonglong2(ix, iy);
    __syncthreads();
    if (warp == 0) {   // exclusive prefix of the 32 warp totals by one warp; the total in s_w[32]
        const ulonglong2 x = s_w[lane];
        const uint64_t px = warp_incl_scan(x.x, lane), py = warp_incl_scan(x.y, lane);
        __syncwarp();
        s_w[lane] = make_ulonglong2(px - x.x, py - x.y);
        if (lane == 31) s_w[kLsWarps] = make_ulonglong2(px, py);
    }
    __syncthreads();
    const ulonglong2 o = s_w[warp], t = s_w[kLsWarps];
    __syncthreads();
    off = make_ulonglong2(o.x + ix - v.x, o.y + iy - v.y);
    return t;
}

// Two-value exclusive prefix over the CTA's warps (warp totals t) and over the cluster's CTAs.
// Returns the offset of the calling warp within the cluster round; *round_total = the round's total.
__device__ __forceinline__ ulonglong2 cluster_offsets(ulonglong2 t, ulonglong2* s_w, ulonglong2* s_tot,
                                                      ulonglong2* s_base, ulonglong2& round_total)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_w[warp] = t;
    __syncthreads();
    if (warp == 0) {
        const ulonglong2 v = s_w[lane];
        const uint64_t ix = warp_incl_scan(v.x, lane), iy = warp_incl_scan(v.y, lane);
        s_w[lane] = make_ulonglong2(ix - v.x, iy - v.y);
        if (lane == 31) *s_tot = make_ulonglong2(ix, iy);
    }
    cluster.sync();                                  // every CTA's total is visible cluster-wide
    if (warp == 0) {
        const unsigned rank = cluster.block_rank(), nc = cluster.num_blocks();
        ulonglong2 v = make_ulonglong2(0ull, 0ull);
        if ((unsigned)lane < nc) v = *cluster.map_shared_rank(s_tot, lane);
        const uint64_t px = warp_sum((unsigned)lane < rank ? v.x : 0ull);
        const uint64_t py = warp_sum((unsigned)lane < rank ? v.y : 0ull);
        const uint64_t tx = warp_sum(v.x), ty = warp_sum(v.y);
        if (lane == 0) { s_base[0] = make_ulonglong2(px, py); s_base[1] = make_ulonglong2(tx, ty); }
    }
    __syncthreads();
    const ulonglong2 w = s_w[warp], cb = s_base[0];
    round_total = s_base[1];
    __syncthreads();
    return make_ulonglong2(cb.x + w.x, cb.y + w.y);
}

// A_all: born mass of every shard (band contexts, gathered after k_cells), or nullptr (whole grid): the
// slots of the band's cells are allocated on the GLOBAL born-mass CDF (prefix of the shards below).
__global__ __launch_bounds__(kLsThreads) void k_list_scan(StageList Ls, CellList L, BlockTotals bt, uint32_t nblk,
                                                          uint32_t chunk, uint32_t* __restrict__ cell2list,
                                                          const uint64_t* __restrict__ A_all,
                                                          DevScalars* sc, FilterConst fc, int64_t k)
{
    PDL_ENTER();
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ uint32_t s_cnt0[kMaxCellBlocks + 1];
    __shared__ ulonglong2 s_w[kLsWarps + 1];
    __shared__ ulonglong2 s_tot[2];
    __shared__ ulonglong2 s_base[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster.block_rank(), nc = cluster.num_blocks();
    // chunk offsets (exclusive prefix of the staged counts) and the grand totals n_in, A -- every CTA
    // forms them itself from k_cells' per-chunk totals (nblk <= 4096: four per thread)
    uint32_t Lc;
    uint64_t A, N, Apre = 0;
    {
        constexpr int kI = (kMaxCellBlocks + kLsThreads - 1) / kLsThreads;
        uint32_t cv[kI];
        uint32_t cs = 0;
        uint64_t as = 0, ns = 0;
#pragma unroll
        for (int i = 0; i < kI; ++i) {
            const uint32_t b = tid * kI + i;
            cv[i] = b < nblk ? bt.cnt[b] : 0u;
            cs += cv[i];
            if (b < nblk) { as += bt.rb0[b]; ns += bt.n0[b]; }
        }
        ulonglong2 off;
        ulonglong2 tot = cta_excl_scan2(make_ulonglong2(cs, 0ull), s_w, off);
        uint32_t run = (uint32_t)off.x;
#pragma unroll
        for (int i = 0; i < kI; ++i) {
            const uint32_t b = tid * kI + i;
            if (b < nblk) s_cnt0[b] = run;
            run += cv[i];
        }
        Lc = (uint32_t)tot.x;
        const ulonglong2 t2 = cta_excl_scan2(make_ulonglong2(as, ns), s_w, off);
        A = t2.x;
        N = t2.y;
        if (A_all) {                                        // global born-mass CDF over the shards
            uint64_t pre = 0, tot_all = 0;
            for (uint32_t r = 0; r < fc.world; ++r) { if (r < fc.rank) pre += A_all[r]; tot_all += A_all[r]; }
            Apre = pre;
            A = tot_all;
        }
        if (tid == 0) {
            s_cnt0[nblk] = Lc;
            if (rank == 0) { sc->Lc = Lc; sc->A = A; sc->n_in = N; }
        }
    }
    const uint64_t nu_b = fc.nu_b;
    const double rcpA = A ? 1.0 / (double)A : 0.0;
    __syncthreads();
    const uint32_t cap = nc * kLsThreads * kLsItems;
    ulonglong2 carry1 = make_ulonglong2(0ull, Apre), carry2 = make_ulonglong2(0ull, 0ull);
    for (uint32_t r0 = 0; r0 < Lc; r0 += cap) {
        const uint32_t gw = r0 + rank * (kLsThreads * kLsItems) + warp * (32 * kLsItems) + lane;   // + 32 i
        uint32_t c[kLsItems], n[kLsItems], npv[kLsItems];
        uint64_t Rb[kLsItems], Rp[kLsItems], X[kLsItems];
        float rho[kLsItems];
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const uint32_t g = gw + 32 * i;
            c[i] = 0; n[i] = 0; npv[i] = 0; Rb[i] = 0; Rp[i] = 0; rho[i] = 0.0f;
            if (g < Lc) {   // staged position: chunk b = last with cnt0[b] <= g
                uint32_t lo = 0, hi = nblk;
                while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (s_cnt0[m] <= g) lo = m; else hi = m; }
                const uint32_t si = lo * chunk + (g - s_cnt0[lo]);
                c[i] = Ls.c[si]; n[i] = Ls.n[si]; npv[i] = Ls.np[si];
                Rb[i] = Ls.Rb[si]; Rp[i] = Ls.Rp[si]; rho[i] = Ls.rho_p[si];
            }
            X[i] = (uint64_t)n[i] | ((uint64_t)npv[i] << 32);
        }
        uint64_t exX[kLsItems], exB[kLsItems];
        const uint64_t wX = warp_excl_items<kLsItems>(X, exX);
        const uint64_t wB = warp_excl_items<kLsItems>(Rb, exB);
        ulonglong2 tot1;
        const ulonglong2 off1 = cluster_offsets(make_ulonglong2(wX, wB), s_w, &s_tot[0], s_base, tot1);
        const ulonglong2 base1 = make_ulonglong2(carry1.x + off1.x, carry1.y + off1.y);
        uint64_t J[kLsItems], its[kLsItems], sp[kLsItems], bbv[kLsItems];
        uint32_t nbv[kLsItems], rbv[kLsItems];
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const bool ok = gw + 32 * i < Lc;
            const uint64_t Ax = base1.y + exB[i];   // A_{c-1}
            sp[i] = ok ? slot_of(Ax, A, nu_b, rcpA) : 0ull;
            const uint64_t s_next = Rb[i] ? slot_of(Ax + Rb[i], A, nu_b, rcpA) : sp[i];
            nbv[i] = (uint32_t)(s_next - sp[i]);
            J[i] = ok ? Rp[i] + (nbv[i] ? Rb[i] : 0ull) : 0ull;
            its[i] = (nbv[i] + kItem - 1) / kItem;
        }
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const uint32_t g = gw + 32 * i;
            if (g >= Lc) continue;
            const uint64_t x0 = base1.x + exX[i];
            L.c[g] = c[i]; L.n[g] = n[i]; L.Rp[g] = Rp[i]; L.rho_p[g] = rho[i];
            L.np[g] = npv[i]; L.ps[g] = (uint32_t)(x0 >> 32); L.pfill[g] = 0u;
            L.start[g] = (uint32_t)x0;
            L.sb[g] = (uint32_t)sp[i];
            L.nb[g] = nbv[i];
            uint32_t rem = 0;
            L.bp[g] = n[i] ? divmod53(Rp[i], n[i], rem) : 0ull;
            L.rp[g] = rem;
            rem = 0;
            bbv[i] = nbv[i] ? divmod53(Rb[i], nbv[i], rem) : 0ull;
            rbv[i] = rem;
            L.bb[g] = bbv[i];
            L.rb[g] = rem;
            cell2list[c[i]] = g;
        }
        uint64_t exJ[kLsItems], exI[kLsItems];
        const uint64_t wJ = warp_excl_items<kLsItems>(J, exJ);
        const uint64_t wI = warp_excl_items<kLsItems>(its, exI);
        ulonglong2 tot2;
        const ulonglong2 off2 = cluster_offsets(make_ulonglong2(wJ, wI), s_w, &s_tot[1], s_base, tot2);
        const ulonglong2 base2 = make_ulonglong2(carry2.x + off2.x, carry2.y + off2.y);
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const uint32_t g = gw + 32 * i;
            if (g >= Lc) continue;
            const uint64_t P = base2.x + exJ[i];
            const uint32_t it0 = (uint32_t)(base2.y + exI[i]);
            L.P[g] = P;
            L.it[g] = it0;
            if (nbv[i]) L.brec[g] = BirthRec{P + Rp[i], bbv[i], c[i], nbv[i], (uint32_t)sp[i], rbv[i]};
            if (g == Lc - 1) {   // the list's last entry publishes the totals (this context's W)
                sc->W = P + J[i];
                sc->n_items = it0 + (uint32_t)its[i];
                sc->s_total = A ? (uint64_t)fc.nu_b : 0ull;
                sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
            }
        }
        carry1.x += tot1.x; carry1.y += tot1.y;
        carry2.x += tot2.x; carry2.y += tot2.y;
    }
    if (Lc == 0 && rank == 0 && tid == 0) {   // empty list (A-26)
        sc->W = 0; sc->n_items = 0; sc->s_total = A ? (uint64_t)fc.nu_b : 0ull;
        sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
    }
    cluster.sync();   // no CTA leaves while another may still read its shared memory
}

// ------------------------------------------------------------------------------------------------
// The same flat active list for LARGE lists (the exact PHD/MIB filter stages every cell: r_b > 0
// everywhere), grid-wide instead of one cluster: the tiles are k_cells' chunks, whose pair-1 totals
// (entries, n_c, runs, R_b) k_cells already wrote (BlockTotals).
//   k_ls_prefix1  (1 block): exclusive prefixes of the chunk totals; Lc, n_in, A
//   k_ls_chunks1  (chunk per block): local scans + chunk prefix -> start, ps, A_c -> slots, split, J, items
//                 -> the list entries; chunk totals of (J, items)
//   k_ls_prefix2  (1 block): exclusive prefixes of (J, items)
//   k_ls_chunks2  (chunk per block): local scans of (J, items) -> P, it; the last entry publishes W, U
// Integer sums, so every prefix equals the cluster kernel's (and the oracle's) exactly.
struct WideScan {
    uint32_t* pcnt; uint64_t* pn; uint32_t* pnp; uint64_t* prb;   // chunk prefixes, pair 1
    uint64_t* tJ; uint32_t* tit;                                  // chunk totals, pair 2
    uint64_t* pJ; uint32_t* pit;                                  // chunk prefixes, pair 2
};

// A_all: born mass of every shard (band contexts) or nullptr: the born-mass CDF then starts at the
// prefix of the shards below and A is the global total (as in k_list_scan).
__global__ __launch_bounds__(1024) void k_ls_prefix1(BlockTotals bt, uint32_t nblk, WideScan ws,
                                                     DevScalars* sc, const uint64_t* __restrict__ A_all,
                                                     FilterConst fc)
{
    PDL_ENTER();
    __shared__ uint64_t s_w[33];
    constexpr int kI = (kMaxCellBlocks + 1023) / 1024;
    const int tid = threadIdx.x;
    uint64_t c[kI], n[kI], p[kI], r[kI], sc_ = 0, sn = 0, sp = 0, sr = 0;
#pragma unroll
    for (int i = 0; i < kI; ++i) {
        const uint32_t b = tid * kI + i;
        const bool ok = b < nblk;
        c[i] = ok ? bt.cnt[b] : 0u; n[i] = ok ? bt.n0[b] : 0ull; p[i] = ok ? bt.np0[b] : 0u; r[i] = ok ? bt.rb0[b] : 0ull;
        sc_ += c[i]; sn += n[i]; sp += p[i]; sr += r[i];
    }
    uint64_t tc, tn, tp, tr;
    uint64_t oc = block_excl_scan<uint64_t, 32>(sc_, s_w, tc);
    uint64_t on = block_excl_scan<uint64_t, 32>(sn, s_w, tn);
    uint64_t op = block_excl_scan<uint64_t, 32>(sp, s_w, tp);
    uint64_t orb = block_excl_scan<uint64_t, 32>(sr, s_w, tr);
    if (A_all) {                                   // global born-mass CDF over the shards
        uint64_t pre = 0, tot = 0;
        for (uint32_t r = 0; r < fc.world; ++r) { if (r < fc.rank) pre += A_all[r]; tot += A_all[r]; }
        orb += pre;
        tr = tot;
    }
#pragma unroll
    for (int i = 0; i < kI; ++i) {
        const uint32_t b = tid * kI + i;
        if (b < nblk) { ws.pcnt[b] = (uint32_t)oc; ws.pn[b] = on; ws.pnp[b] = (uint32_t)op; ws.prb[b] = orb; }
        oc += c[i]; on += n[i]; op += p[i]; orb += r[i];
    }
    if (tid == 0) { sc->Lc = (uint32_t)tc; sc->A = tr; sc->n_in = tn; }
}

__global__ __launch_bounds__(256) void k_ls_chunks1(StageList Ls, CellList L, BlockTotals bt, uint32_t chunk,
                                                    uint32_t* __restrict__ cell2list, WideScan ws,
                                                    const DevScalars* sc, FilterConst fc, uint32_t dense)
{
    PDL_ENTER();
    __shared__ uint64_t s_w[9];
    const uint32_t b = blockIdx.x, m = bt.cnt[b];
    const uint64_t A = scrd(sc->A), nu_b = fc.nu_b;
    const double rcpA = A ? 1.0 / (double)A : 0.0;
    uint64_t carryX = ((uint64_t)ws.pnp[b] << 32) | ws.pn[b], carryB = ws.prb[b], sJ = 0, sI = 0;
    for (uint32_t j0 = 0; j0 < m; j0 += 256) {             // block-uniform trip count
        const uint32_t j = j0 + threadIdx.x;
        const bool ok = j < m;
        const uint32_t si = b * chunk + j;
        uint32_t c = 0, n = 0, npv = 0;
        uint64_t Rp = 0, Rb = 0;
        float rho = 0.0f;
        if (ok) {
            n = Ls.n[si]; npv = Ls.np[si]; Rp = Ls.Rp[si]; Rb = Ls.Rb[si];
            if (dense) c = si;                               // (entry = cell; c and rho_p are in place already)
            else { c = Ls.c[si]; rho = Ls.rho_p[si]; }
        }
        const uint64_t X = (uint64_t)n | ((uint64_t)npv << 32);
        uint64_t tX, tB;
        const uint64_t exX = block_excl_scan<uint64_t, 8>(X, s_w, tX);
        const uint64_t exB = block_excl_scan<uint64_t, 8>(Rb, s_w, tB);
        if (ok) {
            const uint32_t g = ws.pcnt[b] + j;
            const uint64_t x0 = carryX + exX, Ax = carryB + exB;
            const uint64_t sp = slot_of(Ax, A, nu_b, rcpA);
            const uint64_t s_next = Rb ? slot_of(Ax + Rb, A, nu_b, rcpA) : sp;
            const uint32_t nbv = (uint32_t)(s_next - sp);
            if (!dense) {   // (dense cycles: k_cells staged every cell in place, entry g = cell c = si)
                L.c[g] = c; L.n[g] = n; L.Rp[g] = Rp; L.rho_p[g] = rho; L.np[g] = npv;
                cell2list[c] = g;
            }
            DOG_ASSERT(!dense || g == si);
            L.ps[g] = (uint32_t)(x0 >> 32); L.pfill[g] = 0u;
            L.start[g] = (uint32_t)x0;
            L.sb[g] = (uint32_t)sp;
            L.nb[g] = nbv;
            uint32_t rem = 0;
            L.bp[g] = n ? divmod53(Rp, n, rem) : 0ull;
            L.rp[g] = rem;
            rem = 0;
            L.bb[g] = nbv ? divmod53(Rb, nbv, rem) : 0ull;
            L.rb[g] = rem;
            sJ += Rp + (nbv ? Rb : 0ull);
            sI += (nbv + kItem - 1) / kItem;
        }
        carryX += tX; carryB += tB;
    }
    uint64_t tJ, tI;
    block_excl_scan<uint64_t, 8>(sJ, s_w, tJ);
    block_excl_scan<uint64_t, 8>(sI, s_w, tI);
    if (threadIdx.x == 0) { ws.tJ[b] = tJ; ws.tit[b] = (uint32_t)tI; }
}

__global__ __launch_bounds__(1024) void k_ls_prefix2(uint32_t nblk, WideScan ws)
{
    PDL_ENTER();
    __shared__ uint64_t s_w[33];
    constexpr int kI = (kMaxCellBlocks + 1023) / 1024;
    const int tid = threadIdx.x;
    uint64_t J[kI], I[kI], sJ = 0, sI = 0;
#pragma unroll
    for (int i = 0; i < kI; ++i) {
        const uint32_t b = tid * kI + i;
        J[i] = b < nblk ? ws.tJ[b] : 0ull; I[i] = b < nblk ? ws.tit[b] : 0u;
        sJ += J[i]; sI += I[i];
    }
    uint64_t tJ, tI;
    uint64_t oJ = block_excl_scan<uint64_t, 32>(sJ, s_w, tJ);
    uint64_t oI = block_excl_scan<uint64_t, 32>(sI, s_w, tI);
#pragma unroll
    for (int i = 0; i < kI; ++i) {
        const uint32_t b = tid * kI + i;
        if (b < nblk) { ws.pJ[b] = oJ; ws.pit[b] = (uint32_t)oI; }
        oJ += J[i]; oI += I[i];
    }
}

__global__ __launch_bounds__(256) void k_ls_chunks2(CellList L, BlockTotals bt, WideScan ws,
                                                    DevScalars* sc, FilterConst fc, int64_t k)
{
    PDL_ENTER();
    __shared__ uint64_t s_w[9];
    const uint32_t b = blockIdx.x, m = bt.cnt[b];
    const uint32_t Lc = scrd(sc->Lc);
    const uint64_t A = scrd(sc->A);
    uint64_t carryJ = ws.pJ[b], carryI = ws.pit[b];
    for (uint32_t j0 = 0; j0 < m; j0 += 256) {
        const uint32_t j = j0 + threadIdx.x;
        const bool ok = j < m;
        const uint32_t g = ws.pcnt[b] + j;
        uint64_t J = 0, I = 0, Rpg = 0, bbg = 0;
        uint32_t nbv = 0, rbg = 0;
        if (ok) {
            nbv = L.nb[g];
            Rpg = L.Rp[g];
            if (nbv) { bbg = L.bb[g]; rbg = L.rb[g]; }
            J = Rpg + (nbv ? bbg * nbv + rbg : 0ull);                // R_p + gated R_b = bb nb + rb
            I = (nbv + kItem - 1) / kItem;
        }
        uint64_t tJ, tI;
        const uint64_t eJ = block_excl_scan<uint64_t, 8>(J, s_w, tJ);
        const uint64_t eI = block_excl_scan<uint64_t, 8>(I, s_w, tI);
        if (ok) {
            const uint64_t P = carryJ + eJ;
            const uint32_t it0 = (uint32_t)(carryI + eI);
            L.P[g] = P;
            L.it[g] = it0;
            if (nbv) L.brec[g] = BirthRec{P + Rpg, bbg, L.c[g], nbv, L.sb[g], rbg};
            if (g == Lc - 1) {
                sc->W = P + J;
                sc->n_items = it0 + (uint32_t)I;
                sc->s_total = A ? (uint64_t)fc.nu_b : 0ull;
                sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
            }
        }
        carryJ += tJ; carryI += tI;
    }
    if (Lc == 0 && b == 0 && threadIdx.x == 0) {   // empty list (A-26)
        sc->W = 0; sc->n_items = 0; sc->s_total = A ? (uint64_t)fc.nu_b : 0ull;
        sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
    }
}

}  // namespace dog
