// dog_cells.cuh -- per-cell stages of the cycle (Alg. 3, Alg. 5 slot allocation, Alg. 7 joint CDF).
//
// k_cells: one pass over the grid.  For every cell: n_c (from k_predict's counts), S_c = n_c w_pred
// (Eq. 61, exact), m_p = min(S_c, occ_max) (Eq. 17), m_Fp = min(alpha m_F, 1 - m_p) (Eq. 62),
// Dempster update (Eq. 63), birth split (Eqs. 67-68), fixed-point masses (A-23) and the readouts.
// Cells holding particles or receiving born mass ("active" cells, typically ~1 % of the grid) are
// appended, in cell order, to a compact list through a decoupled look-back; every later stage works
// on that list instead of the whole grid.
//
// k_list_scan: one pass over the active list: prefix of n_c (first sorted slot of each cell), prefix
// of R_b (born-mass CDF) -> exact slot allocation s_c = floor((2 nu_b A_c + A) / (2A)) (A-15), the
// gated joint mass J_c = R_p + [n_b > 0] R_b and its exclusive prefix P_c (the joint CDF in
// cell-interleaved order, A-25), the per-cell even-split parameters, W, w_bar (Eq. 57) and U.
#pragma once
#include <cstdint>
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {

struct CellList {           // SoA, capacity C
    uint32_t* c;            // cell index
    uint32_t* n;            // persistent particles n_c
    uint64_t* Rp;           // floor(rho_p 2^40) (0 if n_c = 0)
    uint64_t* Rb;           // floor(rho_b 2^40) if m_zO > 0 else 0
    float* rho_p;           // f32 rho_p (moments denominator)
    uint32_t* start;        // first cell-sorted slot of the cell          (k_list_scan)
    uint32_t* sb;           // first birth slot of the cell                 (k_list_scan)
    uint32_t* nb;           // birth slots of the cell                      (k_list_scan)
    uint64_t* P;            // exclusive joint prefix P_c                   (k_list_scan)
    uint64_t* bp;           // R_p / n_c        (even split of R_p)         (k_list_scan)
    uint32_t* rp;           // R_p mod n_c
    uint64_t* bb;           // R_b / n_b
    uint32_t* rb;           // R_b mod n_b
};

__device__ __forceinline__ uint64_t fx40(float m)
{
    return (m > 0.0f) ? __double2ull_rz(__dmul_rn((double)m, 1099511627776.0)) : 0ull;
}

struct CellOut {
    uint32_t n;
    float S, mO, mF, rp, rb;
    uint64_t Rp, Rb;
    bool bad;
};

// Alg. 3 for one cell, canonical operation order of DESIGN.md 3.2 (bit-identical to the oracle).
__device__ __forceinline__ CellOut cell_math(uint32_t n, float m_free, float2 z, float w_pred, float alpha,
                                             const FilterConst& fc)
{
    CellOut o;
    o.n = n;
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
        o.mO = __fdiv_rn(__fadd_rn(__fmul_rn(aO, bO), __fadd_rn(__fmul_rn(aO, bW), __fmul_rn(aW, bO))), oneK);
        o.mF = __fdiv_rn(__fadd_rn(__fmul_rn(aF, bF), __fadd_rn(__fmul_rn(aF, bW), __fmul_rn(aW, bF))), oneK);
    }
    const float q = __fmul_rn(fc.p_b, __fsub_rn(1.0f, m_p));               // Eqs. 67-68 (A-11)
    const float den = __fadd_rn(m_p, q);
    o.rb = den > 0.0f ? __fdiv_rn(__fmul_rn(o.mO, q), den) : 0.0f;
    o.rp = __fsub_rn(o.mO, o.rb);
    o.Rp = n > 0 ? fx40(o.rp) : 0ull;                                      // A-23
    o.Rb = z.x > 0.0f ? fx40(o.rb) : 0ull;                                 // P:1197 gate (A-13)
    return o;
}

constexpr int kCellThreads = 256, kCellItems = 4, kCellTile = kCellThreads * kCellItems;

struct CellDebug { float* rho_p; float* rho_b; uint64_t* Rp; uint64_t* Rb; };

// Striped tile: item i of thread t is cell tile*1024 + i*256 + t, so each warp touches 32
// consecutive cells per item (coalesced) and one 32-bit word of the moments-valid bitmask.  All loads
// of a tile are issued before any dependent work; results stay in registers across the look-back.
__global__ __launch_bounds__(kCellThreads) void k_cells(
    uint32_t* __restrict__ counts, float* __restrict__ m_free, const float2* __restrict__ meas,
    float* __restrict__ occ, float* __restrict__ free_out, float2* __restrict__ mean, float* __restrict__ cov,
    uint32_t* __restrict__ mvalid, CellDebug dbg, CellList L, uint32_t* __restrict__ cell2list,
    uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ status, DevScalars* __restrict__ sc,
    FilterConst fc, float alpha)
{
    __shared__ uint32_t s_cnt[kCellItems][kCellThreads / 32];
    __shared__ uint32_t s_tile, s_excl;
    __shared__ uint64_t s_A[8];
    __shared__ uint32_t s_bad[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t base = tile * kCellTile;
    const float w_pred = sc->w_pred;
    const uint32_t lt = (1u << lane) - 1u;

    uint32_t n[kCellItems], prev[kCellItems];
    float mf[kCellItems];
    float2 z[kCellItems];
#pragma unroll
    for (int i = 0; i < kCellItems; ++i) {
        const uint32_t c = base + i * kCellThreads + tid;
        const bool valid = c < fc.C;
        n[i] = valid ? counts[c] : 0u;
        mf[i] = valid ? m_free[c] : 0.0f;
        z[i] = valid ? meas[c] : make_float2(0.0f, 0.0f);
        const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
        prev[i] = (lane == 0 && (word << 5) < fc.C) ? mvalid[word] : 0u;
    }
    CellOut o[kCellItems];
    uint32_t abal[kCellItems];
    uint64_t A_loc = 0;
    uint32_t bad_loc = 0;
#pragma unroll
    for (int i = 0; i < kCellItems; ++i) {
        const uint32_t c = base + i * kCellThreads + tid;
        const bool valid = c < fc.C;
        o[i] = cell_math(n[i], mf[i], z[i], w_pred, alpha, fc);
        const bool vnow = valid && o[i].n > 0 && o[i].rp > 0.0f && o[i].S > 0.0f;
        const uint32_t bal = __ballot_sync(0xffffffffu, vnow);
        const uint32_t pw = __shfl_sync(0xffffffffu, prev[i], 0);
        const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
        if (valid) {
            occ[c] = o[i].mO;
            free_out[c] = o[i].mF;
            m_free[c] = o[i].mF;                    // Alg. 3 store_values
            if (n[i]) counts[c] = 0u;               // ready for the next cycle's k_predict
            if (!vnow && ((pw >> lane) & 1u)) {     // moments were reported last cycle: clear (A-18)
                mean[c] = make_float2(0.0f, 0.0f);
                cov[3 * (size_t)c] = 0.0f; cov[3 * (size_t)c + 1] = 0.0f; cov[3 * (size_t)c + 2] = 0.0f;
            }
            if (dbg.rho_p) {
                dbg.rho_p[c] = o[i].rp; dbg.rho_b[c] = o[i].rb; dbg.Rp[c] = o[i].Rp; dbg.Rb[c] = o[i].Rb;
            }
            A_loc += o[i].Rb;
            bad_loc += o[i].bad ? 1u : 0u;
        }
        if (lane == 0 && (word << 5) < fc.C && bal != pw) mvalid[word] = bal;
        const bool act = valid && (o[i].n > 0 || o[i].Rb > 0);
        abal[i] = __ballot_sync(0xffffffffu, act);
        if (lane == 0) s_cnt[i][warp] = __popc(abal[i]);
    }
    __syncthreads();
    // tile-local exclusive offsets in cell order (item-major, then warp), tile total, look-back
    if (warp == 0) {
        const uint32_t v = lane < kCellItems * 8 ? s_cnt[lane >> 3][lane & 7] : 0u;
        const uint32_t incl = warp_incl_scan(v, lane);
        if (lane < kCellItems * 8) s_cnt[lane >> 3][lane & 7] = incl - v;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = lookback_u30(status, tile, total);
        if (lane == 0) {
            s_excl = excl;
            if (tile == gridDim.x - 1) sc->L = excl + total;
        }
    }
    __syncthreads();
    const uint32_t texcl = s_excl;
#pragma unroll
    for (int i = 0; i < kCellItems; ++i) {
        if ((abal[i] >> lane) & 1u) {
            const uint32_t c = base + i * kCellThreads + tid;
            const uint32_t pos = texcl + s_cnt[i][warp] + __popc(abal[i] & lt);
            L.c[pos] = c; L.n[pos] = o[i].n; L.Rp[pos] = o[i].Rp; L.Rb[pos] = o[i].Rb; L.rho_p[pos] = o[i].rp;
            cell2list[c] = pos;
        }
    }
    // device totals (integers: order-independent)
    A_loc = warp_sum(A_loc);
    bad_loc = warp_sum(bad_loc);
    if (lane == 0) { s_A[warp] = A_loc; s_bad[warp] = bad_loc; }
    __syncthreads();
    if (tid == 0) {
        uint64_t A = 0; uint32_t b = 0;
        for (int w = 0; w < kCellThreads / 32; ++w) { A += s_A[w]; b += s_bad[w]; }
        if (A) atomicAdd((unsigned long long*)&sc->A, (unsigned long long)A);
        if (b) atomicAdd(&sc->meas_bad, b);
    }
}

// ------------------------------------------------------------------------------------------------
// exact floor((2 nu_b X + A) / (2A)) for X <= A < 2^64 without a 128-bit division: fp64 estimate,
// then exact integer correction (the quotient is <= nu_b < 2^30).
__device__ __forceinline__ uint64_t slot_of(uint64_t X, uint64_t A, uint64_t nu_b)
{
    if (A == 0) return 0;
    const u128 num = (u128)2 * (u128)nu_b * (u128)X + (u128)A;
    const u128 den = (u128)2 * (u128)A;
    uint64_t q = (uint64_t)floor(fma((double)X / (double)A, (double)nu_b, 0.5));
    while ((u128)q * den > num) --q;
    while ((u128)(q + 1) * den <= num) ++q;
    return q;
}

constexpr int kLsThreads = 256, kLsItems = 8, kLsTile = kLsThreads * kLsItems;

// Persistent CTAs take list tiles in order from an atomic counter until the list is exhausted (the
// list is short: ~1 % of the grid), so no launch depends on the device-resident list length.
__global__ __launch_bounds__(kLsThreads) void k_list_scan(
    CellList L, uint32_t* __restrict__ tile_ctr, LookbackPair lb1, LookbackPair lb2,
    DevScalars* __restrict__ sc, FilterConst fc, int64_t k)
{
    __shared__ uint64_t s_a[kLsThreads / 32 + 1], s_b[kLsThreads / 32 + 1];
    __shared__ uint32_t s_tile;
    __shared__ ulonglong2 s_ex;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t Ln = sc->L;
    const uint64_t A = sc->A;
    const uint64_t nu_b = fc.nu_b;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        __syncthreads();
        const uint32_t b0 = tile * kLsTile;
        if (b0 >= Ln && tile > 0) return;       // tiles are taken in order: the rest lie beyond too
        const uint32_t b = b0 + tid * kLsItems;

        uint32_t n[kLsItems];
        uint64_t Rb[kLsItems], Rp[kLsItems];
        uint64_t ns = 0, rbs = 0;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const bool ok = b + i < Ln;
            n[i] = ok ? L.n[b + i] : 0u;
            Rb[i] = ok ? L.Rb[b + i] : 0ull;
            Rp[i] = ok ? L.Rp[b + i] : 0ull;
            ns += n[i];
            rbs += Rb[i];
        }
        uint64_t tn, trb;
        const uint64_t xn = block_excl_scan<uint64_t, kLsThreads / 32>(ns, s_a, tn);
        const uint64_t xrb = block_excl_scan<uint64_t, kLsThreads / 32>(rbs, s_b, trb);
        if (warp == 0) {
            const ulonglong2 e = lookback_pair(lb1, tile, make_ulonglong2(tn, trb));
            if (tid == 0) s_ex = e;
        }
        __syncthreads();
        uint64_t start = s_ex.x + xn;
        uint64_t Ax = s_ex.y + xrb;             // A_{c-1}
        uint64_t s_prev = slot_of(Ax, A, nu_b);
        uint64_t J[kLsItems];
        uint64_t js = 0;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            Ax += Rb[i];
            const uint64_t s = Rb[i] ? slot_of(Ax, A, nu_b) : s_prev;
            const uint32_t nbv = (uint32_t)(s - s_prev);
            if (b + i < Ln) {
                L.start[b + i] = (uint32_t)start;
                L.sb[b + i] = (uint32_t)s_prev;
                L.nb[b + i] = nbv;
                L.bp[b + i] = n[i] ? Rp[i] / n[i] : 0ull;
                L.rp[b + i] = n[i] ? (uint32_t)(Rp[i] % n[i]) : 0u;
                L.bb[b + i] = nbv ? Rb[i] / nbv : 0ull;
                L.rb[b + i] = nbv ? (uint32_t)(Rb[i] % nbv) : 0u;
                J[i] = Rp[i] + (nbv ? Rb[i] : 0ull);
            } else {
                J[i] = 0;
            }
            start += n[i];
            js += J[i];
            s_prev = s;
        }
        uint64_t tj;
        const uint64_t xj = block_excl_scan<uint64_t, kLsThreads / 32>(js, s_a, tj);
        if (warp == 0) {
            const ulonglong2 e = lookback_pair(lb2, tile, make_ulonglong2(tj, 0ull));
            if (tid == 0) s_ex = e;
        }
        __syncthreads();
        uint64_t run = s_ex.x + xj;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            if (b + i < Ln) L.P[b + i] = run;
            run += J[i];
        }
        // the thread holding the list's last entry (or tile 0 of an empty list) publishes the totals
        const bool last = Ln == 0 ? (tile == 0 && tid == 0) : (b <= Ln - 1 && Ln - 1 < b + kLsItems);
        if (last) {
            const uint64_t W = run;
            sc->W = W;
            sc->s_total = s_prev;
            sc->n_in = start;
            sc->w_bar = W ? __double2float_rn(__ddiv_rn(__dmul_rn((double)W, 0x1p-40), (double)fc.nu)) : 0.0f;
            sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
        }
        __syncthreads();
    }
}

}  // namespace dog
