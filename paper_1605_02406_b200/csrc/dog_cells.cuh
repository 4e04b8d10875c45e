// dog_cells.cuh -- per-cell stages of the cycle (Alg. 3, Alg. 5 slot allocation, Alg. 7 joint CDF).
//
// k_cells: one pass over the grid.  For every cell: n_c (from k_predict's counts), S_c = n_c w_pred
// (Eq. 61, exact), m_p = min(S_c, occ_max) (Eq. 17), m_Fp = min(alpha m_F, 1 - m_p) (Eq. 62),
// Dempster update (Eq. 63), birth split (Eqs. 67-68), fixed-point masses (A-23) and the readouts.
// Cells holding particles or receiving born mass ("active" cells, typically ~1 % of the grid) are
// staged, in cell order, in their block's segment of a list; every later stage works on that list.
// Each block owns a contiguous chunk of cells, so the list is ordered by (block, position); the last
// block to finish scans the few thousand block totals (no grid-wide look-back chain).
//
// k_list_scan (one block per cell chunk): first sorted slot of each cell (prefix of n_c), born-mass
// CDF A_c (prefix of R_b) -> exact slot allocation s_c = floor((2 nu_b A_c + A) / (2A)) (A-15), the
// gated joint mass J_c = R_p + [n_b > 0] R_b and its prefix (the joint CDF in cell-interleaved order,
// A-25), the even-split parameters, and the work items of k_resample (<= 256 members of one cell).
// Its last block scans the block totals -> joint-CDF offsets, W, w_bar (Eq. 57), U (A-24).
#pragma once
#include <cstdint>
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {

constexpr uint32_t kItem = 256;   // members per k_resample work item

struct CellList {           // SoA staging, capacity nblk * chunk (>= C); entry li belongs to block li / chunk
    uint32_t* c;            // cell index
    uint32_t* n;            // persistent particles n_c
    uint64_t* Rp;           // floor(rho_p 2^40) (0 if n_c = 0)
    uint64_t* Rb;           // floor(rho_b 2^40) if m_zO > 0 else 0
    float* rho_p;           // f32 rho_p (moments denominator)
    uint32_t* start;        // first cell-sorted slot of the cell          (k_list_scan)
    uint32_t* sb;           // first birth slot of the cell (global)        (k_list_scan)
    uint32_t* nb;           // birth slots of the cell                      (k_list_scan)
    uint64_t* Pl;           // block-local exclusive joint prefix           (k_list_scan)
    uint32_t* it;           // block-local exclusive birth work-item prefix (k_list_scan)
    uint64_t* bp;           // R_p / n_c        (even split of R_p)         (k_list_scan)
    uint32_t* rp;           // R_p mod n_c
    uint64_t* bb;           // R_b / n_b
    uint32_t* rb;           // R_b mod n_b
    uint32_t* np;           // runs ("pairs") of the cell over the sort tiles   (k_cells)
    uint32_t* ps;           // block-local exclusive prefix of np               (k_list_scan)
    uint32_t* pfill;        // pair-list fill counter                           (k_list_scan resets)
    uint32_t* pdone;        // finished pairs (moments combine)                 (k_list_scan resets)
};

struct BlockTotals {        // one entry per cell chunk
    uint32_t* cnt;          // active cells staged by the block                (k_cells)
    uint64_t* n0;           // sum of n_c over them -> exclusive prefix        (k_cells, last block)
    uint64_t* rb0;          // sum of R_b over them -> exclusive prefix        (k_cells, last block)
    uint64_t* P0;           // sum of J -> exclusive joint prefix of the block  (k_list_scan, last block)
    uint32_t* item0;        // birth work items -> exclusive prefix             (k_list_scan, last block)
    uint32_t* ps0;          // pairs -> exclusive prefix of the block           (k_list_scan, last block)
    uint32_t* s0;           // first birth slot of the block (global)           (k_list_scan)
    uint32_t* done;         // [2] finished-block counters of k_cells / k_list_scan (zeroed per cycle)
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
    o.Rp = n > 0 ? fx40(o.rp) : 0ull;                                      // A-23
    o.Rb = z.x > 0.0f ? fx40(o.rb) : 0ull;                                 // P:1197 gate (A-13)
    return o;
}

constexpr int kCellThreads = 256, kCellItems = 4, kCellIter = kCellThreads * kCellItems;   // 1024 cells
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

// Block b owns cells [b chunk, (b+1) chunk), 1024 per iteration; item i of thread t in an iteration
// is cell base + i*256 + t (coalesced; one warp = one 32-bit word of the moments-valid bitmask).
__global__ __launch_bounds__(kCellThreads) void k_cells(
    uint32_t* __restrict__ counts, uint32_t* __restrict__ npairs, float* __restrict__ m_free, const float2* __restrict__ meas,
    float* __restrict__ occ, float* __restrict__ free_out, float2* __restrict__ mean, float* __restrict__ cov,
    uint32_t* __restrict__ mvalid, CellDebug dbg, CellList L, uint32_t* __restrict__ cell2list,
    BlockTotals bt, uint32_t chunk, DevScalars* __restrict__ sc, FilterConst fc, float alpha)
{
    __shared__ uint32_t s_cnt[kCellItems][kCellThreads / 32];
    __shared__ uint32_t s_run;
    __shared__ uint64_t s_A[9], s_N[9];
    __shared__ uint32_t s_bad[8];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const float w_pred = sc->w_pred;
    const uint32_t c0 = blockIdx.x * chunk;
    const uint32_t c1 = min(c0 + chunk, fc.C);
    const uint32_t lbase = blockIdx.x * chunk;
    if (tid == 0) s_run = 0;

    uint64_t A_loc = 0, N_loc = 0;
    uint32_t bad_loc = 0;
    for (uint32_t base = c0; base < c1; base += kCellIter) {
        uint32_t n[kCellItems], prev[kCellItems];
        float mf[kCellItems];
        float2 z[kCellItems];
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            const uint32_t c = base + i * kCellThreads + tid;
            const bool valid = c < c1;
            n[i] = valid ? counts[c] : 0u;
            mf[i] = valid ? m_free[c] : 0.0f;
            z[i] = valid ? meas[c] : make_float2(0.0f, 0.0f);
            const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
            prev[i] = (lane == 0 && (word << 5) < c1) ? mvalid[word] : 0u;
        }
        CellOut o[kCellItems];
        uint32_t abal[kCellItems];
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            const uint32_t c = base + i * kCellThreads + tid;
            const bool valid = c < c1;
            o[i] = cell_math(n[i], mf[i], z[i], w_pred, alpha, fc);
            const bool vnow = valid && o[i].n > 0 && o[i].rp > 0.0f && o[i].S > 0.0f;
            const uint32_t bal = __ballot_sync(0xffffffffu, vnow);
            const uint32_t pw = __shfl_sync(0xffffffffu, prev[i], 0);
            const uint32_t word = (base + i * kCellThreads + warp * 32) >> 5;
            if (valid) {
                occ[c] = o[i].mO;
                free_out[c] = o[i].mF;
                m_free[c] = o[i].mF;                    // Alg. 3 store_values
                if (n[i]) counts[c] = 0u;               // ready for the next cycle's k_tilesort
                if (!vnow && ((pw >> lane) & 1u)) {     // moments were reported last cycle: clear (A-18)
                    mean[c] = make_float2(0.0f, 0.0f);
                    cov[3 * (size_t)c] = 0.0f; cov[3 * (size_t)c + 1] = 0.0f; cov[3 * (size_t)c + 2] = 0.0f;
                }
                if (dbg.rho_p) {
                    dbg.rho_p[c] = o[i].rp; dbg.rho_b[c] = o[i].rb; dbg.Rp[c] = o[i].Rp; dbg.Rb[c] = o[i].Rb;
                }
                bad_loc += o[i].bad ? 1u : 0u;
            }
            if (lane == 0 && (word << 5) < c1 && bal != pw) mvalid[word] = bal;
            const bool act = valid && (o[i].n > 0 || o[i].Rb > 0);
            abal[i] = __ballot_sync(0xffffffffu, act);
            if (lane == 0) s_cnt[i][warp] = __popc(abal[i]);
        }
        __syncthreads();
        if (warp == 0) {   // exclusive offsets in cell order (item-major, then warp) + running total
            const uint32_t v = lane < kCellItems * 8 ? s_cnt[lane >> 3][lane & 7] : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            const uint32_t run = s_run;
            if (lane < kCellItems * 8) s_cnt[lane >> 3][lane & 7] = run + incl - v;
            __syncwarp();
            if (lane == 31) s_run = run + incl;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kCellItems; ++i) {
            if ((abal[i] >> lane) & 1u) {
                const uint32_t c = base + i * kCellThreads + tid;
                const uint32_t li = lbase + s_cnt[i][warp] + __popc(abal[i] & lt);
                L.c[li] = c; L.n[li] = o[i].n; L.Rp[li] = o[i].Rp; L.Rb[li] = o[i].Rb; L.rho_p[li] = o[i].rp;
                uint32_t npc = 0;
                if (o[i].n) { npc = npairs[c]; npairs[c] = 0u; }
                L.np[li] = npc;
                cell2list[c] = li;
                A_loc += o[i].Rb;
                N_loc += o[i].n;
            }
        }
        __syncthreads();
    }
    // block totals (integers: order-independent)
    A_loc = warp_sum(A_loc);
    N_loc = warp_sum(N_loc);
    bad_loc = warp_sum(bad_loc);
    if (lane == 0) { s_A[warp] = A_loc; s_N[warp] = N_loc; s_bad[warp] = bad_loc; }
    __syncthreads();
    if (tid == 0) {
        uint64_t A = 0, N = 0; uint32_t b = 0;
        for (int w = 0; w < kCellThreads / 32; ++w) { A += s_A[w]; N += s_N[w]; b += s_bad[w]; }
        bt.cnt[blockIdx.x] = s_run;
        bt.n0[blockIdx.x] = N;
        bt.rb0[blockIdx.x] = A;
        if (b) atomicAdd(&sc->meas_bad, b);
        __threadfence();
        s_last = atomicAdd(&bt.done[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // the last block: exclusive prefixes of the block totals, grand totals
    __threadfence();
    const uint64_t N = block_prefix_inplace<uint64_t>(bt.n0, gridDim.x, s_N);
    const uint64_t A = block_prefix_inplace<uint64_t>(bt.rb0, gridDim.x, s_A);
    if (tid == 0) { sc->n_in = N; sc->A = A; }
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

__global__ __launch_bounds__(kLsThreads) void k_list_scan(CellList L, BlockTotals bt, uint32_t chunk,
                                                          DevScalars* __restrict__ sc, FilterConst fc, int64_t k)
{
    __shared__ uint64_t s_a[kLsThreads / 32 + 1], s_b[kLsThreads / 32 + 1];
    __shared__ uint32_t s_c[kLsThreads / 32 + 1];
    __shared__ bool s_last;
    const int tid = threadIdx.x;
    const uint32_t blk = blockIdx.x;
    const uint64_t A = sc->A;
    const uint64_t nu_b = fc.nu_b;
    uint64_t start0 = bt.n0[blk], A0 = bt.rb0[blk];
    const uint32_t cnt = bt.cnt[blk];
    const uint32_t lbase = blk * chunk;
    if (tid == 0) bt.s0[blk] = (uint32_t)slot_of(A0, A, nu_b);
    uint64_t J0 = 0;                          // block-local joint prefix
    uint32_t I0 = 0;                          // block-local birth work-item prefix
    uint32_t PS0 = 0;                         // block-local pair prefix
    for (uint32_t t0 = 0; t0 < cnt; t0 += kLsTile) {
        const uint32_t b = t0 + tid * kLsItems;
        uint32_t n[kLsItems], npv[kLsItems];
        uint64_t Rb[kLsItems], Rp[kLsItems];
        uint64_t ns = 0, rbs = 0;
        uint32_t pss = 0;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const bool ok = b + i < cnt;
            n[i] = ok ? L.n[lbase + b + i] : 0u;
            npv[i] = ok ? L.np[lbase + b + i] : 0u;
            Rb[i] = ok ? L.Rb[lbase + b + i] : 0ull;
            Rp[i] = ok ? L.Rp[lbase + b + i] : 0ull;
            ns += n[i];
            rbs += Rb[i];
            pss += npv[i];
        }
        uint32_t tps;
        uint32_t xps = PS0 + block_excl_scan<uint32_t, kLsThreads / 32>(pss, s_c, tps);
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            if (b + i < cnt) L.ps[lbase + b + i] = xps;
            xps += npv[i];
        }
        PS0 += tps;
        uint64_t tn, trb;
        const uint64_t xn = block_excl_scan<uint64_t, kLsThreads / 32>(ns, s_a, tn);
        const uint64_t xrb = block_excl_scan<uint64_t, kLsThreads / 32>(rbs, s_b, trb);
        uint64_t start = start0 + xn;
        uint64_t Ax = A0 + xrb;               // A_{c-1}
        uint64_t s_prev = slot_of(Ax, A, nu_b);
        uint64_t J[kLsItems];
        uint32_t its[kLsItems];
        uint64_t js = 0;
        uint32_t is = 0;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            Ax += Rb[i];
            const uint64_t s = Rb[i] ? slot_of(Ax, A, nu_b) : s_prev;
            const uint32_t nbv = (uint32_t)(s - s_prev);
            if (b + i < cnt) {
                const uint32_t li = lbase + b + i;
                L.start[li] = (uint32_t)start;
                L.sb[li] = (uint32_t)s_prev;
                L.nb[li] = nbv;
                L.bp[li] = n[i] ? Rp[i] / n[i] : 0ull;
                L.rp[li] = n[i] ? (uint32_t)(Rp[i] % n[i]) : 0u;
                L.bb[li] = nbv ? Rb[i] / nbv : 0ull;
                L.rb[li] = nbv ? (uint32_t)(Rb[i] % nbv) : 0u;
                L.pfill[li] = 0u;
                L.pdone[li] = 0u;
                J[i] = Rp[i] + (nbv ? Rb[i] : 0ull);
                its[i] = (nbv + kItem - 1) / kItem;
            } else {
                J[i] = 0;
                its[i] = 0;
            }
            start += n[i];
            js += J[i];
            is += its[i];
            s_prev = s;
        }
        uint64_t tj;
        uint32_t ti;
        const uint64_t xj = block_excl_scan<uint64_t, kLsThreads / 32>(js, s_a, tj);
        const uint32_t xi = block_excl_scan<uint32_t, kLsThreads / 32>(is, s_c, ti);
        uint64_t run = J0 + xj;
        uint32_t irun = I0 + xi;
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            if (b + i < cnt) { L.Pl[lbase + b + i] = run; L.it[lbase + b + i] = irun; }
            run += J[i];
            irun += its[i];
        }
        start0 += tn;
        A0 += trb;
        J0 += tj;
        I0 += ti;
    }
    if (tid == 0) {
        bt.P0[blk] = J0;
        bt.item0[blk] = I0;
        bt.ps0[blk] = PS0;
        __threadfence();
        s_last = atomicAdd(&bt.done[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // the last block: joint-CDF and work-item offsets of the chunks, totals (Eq. 57, A-24, A-26)
    __threadfence();
    const uint64_t W = block_prefix_inplace<uint64_t>(bt.P0, gridDim.x, s_a);
    const uint32_t items = block_prefix_inplace<uint32_t>(bt.item0, gridDim.x, s_c);
    block_prefix_inplace<uint32_t>(bt.ps0, gridDim.x, s_c);
    if (tid == 0) {
        sc->W = W;
        sc->n_items = items;
        sc->s_total = A ? (uint64_t)fc.nu_b : 0ull;
        sc->w_bar = W ? __double2float_rn(__ddiv_rn(__dmul_rn((double)W, 0x1p-40), (double)fc.nu)) : 0.0f;
        sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
    }
}

}  // namespace dog
