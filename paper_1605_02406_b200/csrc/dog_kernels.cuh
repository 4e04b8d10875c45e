// dog_kernels.cuh -- the sm_100a kernels of one DS-PHD/MIB cycle (section VII).
//
// Stage map (paper -> kernel):
//   Alg. 1 predict              -> k_predict      (+ cell counts, radix histograms)
//   Alg. 2 sort + assign        -> k_onesweep x P (stable LSD radix sort of (key, idx))
//                                                 k_scan_counts (counts -> offsets)
//   Alg. 3 occupancy predict/update           -> k_cells        (Eqs. 61-63, 67-68, fixed point)
//   Alg. 4 persistent update    -> implicit: weights are uniform per cell (A-8, A-23)
//   Alg. 5 new-born particles   -> k_scan_joint (slot scan + joint CDF), k_births
//   Alg. 6 moments              -> k_moments + k_moments_fixup (segmented reduction)
//   Alg. 7 resampling           -> k_resample (systematic, exact u64/u128 arithmetic)
//
// Every floating-point expression on the parity path uses explicit round-to-nearest intrinsics in
// the operation order of DESIGN.md section 3 so the CPU oracle reproduces it bit for bit (A-21).
#pragma once
#include <cstdint>
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {

constexpr float kSentinelPos = -1073741824.0f;  // -2^30 cells: empty-world particle (A-19)
constexpr float kMeasSumMax = 0x1.00001p+0f;    // 1 + 2^-20 (= 1.0f + 1e-6f rounded), A-27

// ------------------------------------------------------------------------------------------------
// Alg. 1 -- particle prediction.  Each thread advances 4 consecutive particles (16-byte SoA I/O).
// Also: warp-aggregated per-cell counts n_c (for offsets) and the radix-sort digit histograms.
// ------------------------------------------------------------------------------------------------
constexpr int kPredThreads = 256;
constexpr int kMaxPasses = 4;

__global__ __launch_bounds__(kPredThreads) void k_predict(
    const float4* __restrict__ x, const float4* __restrict__ y, const float4* __restrict__ vx,
    const float4* __restrict__ vy, float4* __restrict__ px, float4* __restrict__ py,
    float4* __restrict__ pvx, float4* __restrict__ pvy, uint4* __restrict__ keys,
    uint32_t* __restrict__ key_dbg, uint32_t* __restrict__ counts, uint32_t* __restrict__ rhist,
    int npass, DevScalars* __restrict__ sc, FilterConst fc, StepArgs a)
{
    __shared__ uint32_t s_hist[kMaxPasses * 256];
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();

    const float w_bar = sc->w_bar;
    const float w_pred = __fmul_rn(fc.p_s, w_bar);      // Eq. 39 (A-3): one scalar
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->w_pred = w_pred;
    const float Wf = (float)fc.W, Hf = (float)fc.H;
    const uint32_t n4 = (fc.nu + 3u) >> 2;
    const int lane = threadIdx.x & 31;

    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g - lane < n4;
         g += gridDim.x * blockDim.x) {
        const bool gv = g < n4;
        float4 X = make_float4(0, 0, 0, 0), Y = X, VX = X, VY = X;
        if (gv) { X = x[g]; Y = y[g]; VX = vx[g]; VY = vy[g]; }
        float xs[4] = {X.x, X.y, X.z, X.w}, ys[4] = {Y.x, Y.y, Y.z, Y.w};
        float vxs[4] = {VX.x, VX.y, VX.z, VX.w}, vys[4] = {VY.x, VY.y, VY.z, VY.w};
        uint32_t ks[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t i = g * 4u + e;
            const Philox4 r = draw(fc.seed, i, a.k, STAGE_PREDICT);
            float n0, n1, n2, n3;
            box_muller(r.r0, r.r1, n0, n1);
            box_muller(r.r2, r.r3, n2, n3);
            // p' = p + T v + xi_p with the OLD velocity (Eq. 14, A-2); v' = v + xi_v
            const float xn = __fmaf_rn(a.s_p, n0, __fmaf_rn(vxs[e], a.Tc, xs[e]));
            const float yn = __fmaf_rn(a.s_p, n1, __fmaf_rn(vys[e], a.Tc, ys[e]));
            vxs[e] = __fmaf_rn(a.s_v, n2, vxs[e]);
            vys[e] = __fmaf_rn(a.s_v, n3, vys[e]);
            xs[e] = xn; ys[e] = yn;
            const bool inside = (xn >= 0.0f) && (xn < Wf) && (yn >= 0.0f) && (yn < Hf);
            const bool valid = gv && i < fc.nu;
            ks[e] = inside ? (uint32_t)__float2int_rz(yn) * (uint32_t)fc.W + (uint32_t)__float2int_rz(xn)
                           : fc.C;                                  // A-4, A-5
            // per-cell counts (sentinel excluded), warp-aggregated
            const uint32_t ck = (valid && inside) ? ks[e] : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, ck);
            if (ck != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&counts[ck], __popc(peers));
            if (valid) {
                for (int p = 0; p < npass; ++p) atomicAdd(&s_hist[p * 256 + ((ks[e] >> (8 * p)) & 255u)], 1u);
                if (key_dbg) key_dbg[i] = ks[e];
            }
        }
        if (gv) {
            px[g] = make_float4(xs[0], xs[1], xs[2], xs[3]);
            py[g] = make_float4(ys[0], ys[1], ys[2], ys[3]);
            pvx[g] = make_float4(vxs[0], vxs[1], vxs[2], vxs[3]);
            pvy[g] = make_float4(vys[0], vys[1], vys[2], vys[3]);
            keys[g] = make_uint4(ks[0], ks[1], ks[2], ks[3]);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&rhist[i], s_hist[i]);
}

// ------------------------------------------------------------------------------------------------
// Alg. 2 -- stable LSD radix sort of (cell key, input index), one kernel per 8-bit digit
// ("onesweep": global digit histograms from k_predict + decoupled look-back across tiles).
// Stability: within a tile, warps own consecutive 512-element slices and rank in order
// (match_any + running per-warp digit counters), so equal digits keep input order (A-6).
// ------------------------------------------------------------------------------------------------
constexpr int kRsThreads = 256, kRsItems = 16, kRsTile = kRsThreads * kRsItems, kRsWarps = 8;
constexpr uint32_t kStAgg = 1u << 30, kStInc = 2u << 30, kStMask = (1u << 30) - 1u;

template <bool FIRST>
__global__ __launch_bounds__(kRsThreads) void k_onesweep(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, const uint32_t* __restrict__ hist,
    uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ status)
{
    __shared__ uint32_t s_keys[kRsTile];
    __shared__ uint32_t s_vals[kRsTile];
    __shared__ uint32_t s_whist[kRsWarps][256];
    __shared__ uint32_t s_gofs[256];
    __shared__ uint32_t s_lstart[256];
    __shared__ uint32_t s_scan[kRsWarps + 1];
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    for (int i = tid; i < kRsWarps * 256; i += kRsThreads) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t base = tile * kRsTile + warp * (kRsItems * 32);
    const uint32_t lt = (1u << lane) - 1u;

    uint32_t k[kRsItems], v[kRsItems], rk[kRsItems];
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        const bool ok = idx < n;
        k[i] = ok ? kin[idx] : 0u;
        v[i] = FIRST ? idx : (ok ? vin[idx] : 0u);
    }
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        const bool ok = idx < n;
        const uint32_t dig = ok ? ((k[i] >> shift) & 255u) : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        const uint32_t r = __popc(peers & lt);
        uint32_t prev = 0;
        if (ok) prev = s_whist[warp][dig];
        __syncwarp();
        if (ok && r == 0) s_whist[warp][dig] = prev + __popc(peers);
        __syncwarp();
        rk[i] = prev + r;
    }
    __syncthreads();
    // per digit (thread = digit): exclusive prefix over warps, tile count
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = run;
        run += c;
    }
    const uint32_t tcount = run;
    // decoupled look-back per digit
    uint32_t* st = status + (size_t)tile * 256 + tid;
    uint32_t excl = 0;
    if (tile == 0) {
        st_relaxed(st, kStInc | tcount);
    } else {
        st_relaxed(st, kStAgg | tcount);
        int j = (int)tile - 1;
        while (true) {
            const uint32_t s = ld_relaxed(status + (size_t)j * 256 + tid);
            if ((s & ~kStMask) == 0) continue;
            excl += s & kStMask;
            if (s & kStInc) break;
            --j;
        }
        st_relaxed(st, kStInc | (excl + tcount));
    }
    uint32_t tot;
    const uint32_t dbase = block_excl_scan<uint32_t, kRsWarps>(hist[tid], s_scan, tot);
    const uint32_t lstart = block_excl_scan<uint32_t, kRsWarps>(tcount, s_scan, tot);
    s_lstart[tid] = lstart;
    s_gofs[tid] = dbase + excl - lstart;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        if (idx < n) {
            const uint32_t dig = (k[i] >> shift) & 255u;
            const uint32_t pos = s_lstart[dig] + s_whist[warp][dig] + rk[i];
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
    }
    __syncthreads();
    const uint32_t tile0 = tile * kRsTile;
    const uint32_t nvalid = n > tile0 ? min((uint32_t)kRsTile, n - tile0) : 0u;
    for (uint32_t p = tid; p < nvalid; p += kRsThreads) {
        const uint32_t key = s_keys[p];
        const uint32_t o = s_gofs[(key >> shift) & 255u] + p;
        kout[o] = key;
        vout[o] = s_vals[p];
    }
}

// ------------------------------------------------------------------------------------------------
// Exclusive scan of per-cell counts -> offsets[0..C] (Alg. 2's start/end indices), single pass
// with decoupled look-back (values < 2^30 packed with a 2-bit status).
// ------------------------------------------------------------------------------------------------
constexpr int kScThreads = 256, kScItems = 16, kScTile = kScThreads * kScItems;

__global__ __launch_bounds__(kScThreads) void k_scan_counts(
    const uint32_t* __restrict__ counts, uint32_t* __restrict__ offsets, uint32_t n,
    uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ status, DevScalars* __restrict__ sc)
{
    __shared__ uint32_t s_scan[kRsWarps + 1];
    __shared__ uint32_t s_tile, s_excl;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t b = tile * kScTile + tid * kScItems;
    uint32_t v[kScItems];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScItems; ++i) {
        v[i] = (b + i < n) ? counts[b + i] : 0u;
        sum += v[i];
    }
    uint32_t total;
    const uint32_t texcl = block_excl_scan<uint32_t, kScThreads / 32>(sum, s_scan, total);
    if (tid == 0) {
        uint32_t excl = 0;
        if (tile == 0) {
            st_relaxed(status, kStInc | total);
        } else {
            st_relaxed(status + tile, kStAgg | total);
            int j = (int)tile - 1;
            while (true) {
                const uint32_t s = ld_relaxed(status + j);
                if ((s & ~kStMask) == 0) continue;
                excl += s & kStMask;
                if (s & kStInc) break;
                --j;
            }
            st_relaxed(status + tile, kStInc | (excl + total));
        }
        s_excl = excl;
    }
    __syncthreads();
    uint32_t run = s_excl + texcl;
#pragma unroll
    for (int i = 0; i < kScItems; ++i) {
        if (b + i < n) offsets[b + i] = run;
        run += v[i];
    }
    if (b < n && b + kScItems >= n) {  // the thread holding the last element writes offsets[n]
        offsets[n] = run;
        sc->n_in = run;
    }
}

// ------------------------------------------------------------------------------------------------
// Alg. 3 -- per-cell occupancy prediction and DS update (one thread per cell).
// S_c = sum of predicted weights (Eq. 61) is n_c * w_pred exactly (uniform weights, A-22);
// m_p = min(S_c, occ_max) (Eq. 17/61, A-7); m_Fp = min(alpha m_F, 1 - m_p) (Eq. 62);
// (m_O, m_F') = m_pred (+) m_z (Eq. 63, A-10); rho_b, rho_p (Eqs. 67-68, A-11); fixed point R_p,
// R_b (A-23) with births gated by m_zO > 0 (A-13).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t fx40(float m)
{
    return (m > 0.0f) ? __double2ull_rz(__dmul_rn((double)m, 1099511627776.0)) : 0ull;
}

__global__ __launch_bounds__(256) void k_cells(
    const uint32_t* __restrict__ offsets, float* __restrict__ m_free, const float2* __restrict__ meas,
    float* __restrict__ occ, float* __restrict__ free_out, float* __restrict__ rho_p_out,
    float* __restrict__ rho_b_dbg, uint64_t* __restrict__ Rp, uint64_t* __restrict__ Rb,
    float2* __restrict__ mean, float* __restrict__ cov, DevScalars* __restrict__ sc, FilterConst fc,
    float alpha)
{
    __shared__ uint64_t s_A[8];
    __shared__ uint32_t s_bad[8];
    const float w_pred = sc->w_pred;
    uint64_t A_loc = 0;
    uint32_t bad_loc = 0;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < fc.C; c += gridDim.x * blockDim.x) {
        const uint32_t n = offsets[c + 1] - offsets[c];
        const float S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));
        const float m_p = fminf(S, fc.occ_max);
        const float m_fp = fminf(__fmul_rn(alpha, m_free[c]), __fsub_rn(1.0f, m_p));
        float2 z = meas[c];
        if (!(z.x >= 0.0f) || !(z.y >= 0.0f) || !(__fadd_rn(z.x, z.y) <= kMeasSumMax)) {
            ++bad_loc;
            z = make_float2(0.0f, 0.0f);
        }
        // Dempster's rule on {O, F, Omega}
        const float aO = m_p, aF = m_fp, aW = __fsub_rn(__fsub_rn(1.0f, aO), aF);
        const float bO = z.x, bF = z.y, bW = __fsub_rn(__fsub_rn(1.0f, bO), bF);
        const float K = __fadd_rn(__fmul_rn(aO, bF), __fmul_rn(aF, bO));
        const float oneK = __fsub_rn(1.0f, K);
        float mO, mF;
        if (oneK <= 0.0f) { mO = bO; mF = bF; }
        else {
            mO = __fdiv_rn(__fadd_rn(__fmul_rn(aO, bO), __fadd_rn(__fmul_rn(aO, bW), __fmul_rn(aW, bO))), oneK);
            mF = __fdiv_rn(__fadd_rn(__fmul_rn(aF, bF), __fadd_rn(__fmul_rn(aF, bW), __fmul_rn(aW, bF))), oneK);
        }
        // birth split (Eqs. 67-68)
        const float q = __fmul_rn(fc.p_b, __fsub_rn(1.0f, m_p));
        const float den = __fadd_rn(m_p, q);
        const float rb = den > 0.0f ? __fdiv_rn(__fmul_rn(mO, q), den) : 0.0f;
        const float rp = __fsub_rn(mO, rb);
        m_free[c] = mF;
        occ[c] = mO;
        free_out[c] = mF;
        rho_p_out[c] = rp;
        if (rho_b_dbg) rho_b_dbg[c] = rb;
        Rp[c] = n > 0 ? fx40(rp) : 0ull;
        const uint64_t rbx = z.x > 0.0f ? fx40(rb) : 0ull;
        Rb[c] = rbx;
        A_loc += rbx;
        if (!(n > 0 && rp > 0.0f && S > 0.0f)) {   // moments undefined: report zeros (A-18)
            mean[c] = make_float2(0.0f, 0.0f);
            cov[3 * (size_t)c] = 0.0f; cov[3 * (size_t)c + 1] = 0.0f; cov[3 * (size_t)c + 2] = 0.0f;
        }
    }
    // block reductions -> device totals (integer, so order-independent)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        A_loc += __shfl_xor_sync(0xffffffffu, A_loc, off);
        bad_loc += __shfl_xor_sync(0xffffffffu, bad_loc, off);
    }
    if (lane == 0) { s_A[warp] = A_loc; s_bad[warp] = bad_loc; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t A = 0; uint32_t b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { A += s_A[w]; b += s_bad[w]; }
        if (A) atomicAdd((unsigned long long*)&sc->A, (unsigned long long)A);
        if (b) atomicAdd(&sc->meas_bad, b);
    }
}

// ------------------------------------------------------------------------------------------------
// Alg. 5 (slot allocation) + Alg. 7 line 4 (joint CDF) in one pass over the cells, two chained
// decoupled look-backs:  A_c = prefix of R_b;  s_c = floor((2 nu_b A_c + A) / (2A)) (A-15);
// n_b(c) = s_c - s_{c-1};  J_c = R_p(c) + [n_b(c) > 0] R_b(c);  P_c = exclusive prefix of J (A-25).
// Outputs sb[c] = s_{c-1} (sb[C] = total slots) and P[c] (P[C] = W).
// ------------------------------------------------------------------------------------------------
constexpr int kJThreads = 256, kJItems = 16, kJTile = kJThreads * kJItems;

__device__ __forceinline__ uint64_t lookback64(uint32_t tile, uint64_t total, uint32_t* flag,
                                               uint64_t* agg, uint64_t* inc)
{
    uint64_t excl = 0;
    if (tile == 0) {
        inc[0] = total;
        st_release(flag, 2u);
    } else {
        agg[tile] = total;
        st_release(flag + tile, 1u);
        int j = (int)tile - 1;
        while (true) {
            const uint32_t f = ld_acquire(flag + j);
            if (f == 0u) continue;
            if (f == 2u) { excl += ld_relaxed64(inc + j); break; }
            excl += ld_relaxed64(agg + j);
            --j;
        }
        inc[tile] = excl + total;
        st_release(flag + tile, 2u);
    }
    return excl;
}

__device__ __forceinline__ uint64_t slot_of(uint64_t X, uint64_t A, uint64_t nu_b)
{
    if (A == 0) return 0;
    return (uint64_t)(((u128)2 * (u128)nu_b * (u128)X + (u128)A) / ((u128)2 * (u128)A));
}

__global__ __launch_bounds__(kJThreads) void k_scan_joint(
    const uint64_t* __restrict__ Rp, const uint64_t* __restrict__ Rb, uint32_t* __restrict__ sb,
    uint64_t* __restrict__ P, uint32_t C, uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ flagA,
    uint64_t* __restrict__ aggA, uint64_t* __restrict__ incA, uint32_t* __restrict__ flagJ,
    uint64_t* __restrict__ aggJ, uint64_t* __restrict__ incJ, DevScalars* __restrict__ sc,
    FilterConst fc, int64_t k)
{
    __shared__ uint64_t s_scan[kJThreads / 32 + 1];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t b = tile * kJTile + tid * kJItems;
    const uint64_t A = sc->A;
    const uint64_t nu_b = fc.nu_b;

    uint64_t rb[kJItems];
    uint64_t sum = 0;
#pragma unroll
    for (int i = 0; i < kJItems; ++i) {
        rb[i] = (b + i < C) ? Rb[b + i] : 0ull;
        sum += rb[i];
    }
    uint64_t total;
    uint64_t texcl = block_excl_scan<uint64_t, kJThreads / 32>(sum, s_scan, total);
    if (tid == 0) s_excl = lookback64(tile, total, flagA, aggA, incA);
    __syncthreads();
    uint64_t Ax = s_excl + texcl;                 // A_{c-1} for the thread's first cell
    uint64_t s_prev = slot_of(Ax, A, nu_b);
    uint64_t J[kJItems];
    uint64_t jsum = 0;
#pragma unroll
    for (int i = 0; i < kJItems; ++i) {
        Ax += rb[i];
        const uint64_t s = rb[i] ? slot_of(Ax, A, nu_b) : s_prev;
        const uint64_t nb = s - s_prev;
        if (b + i < C) {
            sb[b + i] = (uint32_t)s_prev;
            J[i] = Rp[b + i] + (nb ? rb[i] : 0ull);
        } else {
            J[i] = 0;
        }
        jsum += J[i];
        s_prev = s;
    }
    texcl = block_excl_scan<uint64_t, kJThreads / 32>(jsum, s_scan, total);
    if (tid == 0) s_excl = lookback64(tile, total, flagJ, aggJ, incJ);
    __syncthreads();
    uint64_t run = s_excl + texcl;
#pragma unroll
    for (int i = 0; i < kJItems; ++i) {
        if (b + i < C) P[b + i] = run;
        run += J[i];
    }
    if (b < C && b + kJItems >= C) {   // last cell: totals
        sb[C] = (uint32_t)s_prev;
        P[C] = run;
        sc->W = run;
        sc->s_total = s_prev;
        sc->w_bar = run ? __double2float_rn(__ddiv_rn(__dmul_rn((double)run, 0x1p-40), (double)fc.nu)) : 0.0f;
        sc->U = draw(fc.seed, 0u, k, STAGE_RESAMPLE).r0;
    }
}

// ------------------------------------------------------------------------------------------------
// Alg. 6 -- velocity moments of persistent particles (Eqs. 81-84), segmented reduction over the
// cell-sorted particles.  Each warp reduces a range of 256 sorted slots (fp64 shuffle scans);
// segments wholly inside a range are finalised at once, segments crossing ranges are carried
// through head/tail partials and finalised by k_moments_fixup in a fixed order (deterministic).
// ------------------------------------------------------------------------------------------------
constexpr int kMomRange = 256;   // sorted slots per warp
struct MomPartial { double s[5]; };

__device__ __forceinline__ void finalize_cell(uint32_t c, const double* s, const uint32_t* __restrict__ offsets,
                                              const float* __restrict__ rho_p, float w_pred,
                                              float2* __restrict__ mean, float* __restrict__ cov)
{
    const uint32_t n = offsets[c + 1] - offsets[c];
    const float S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));
    const float rp = rho_p[c];
    if (!(rp > 0.0f) || !(S > 0.0f)) return;
    const float w = __fmul_rn(__fdiv_rn(rp, S), w_pred);    // Eq. 71: w' = rho_p / m_p * w_pred
    const double wd = (double)w, rd = (double)rp;
    const double mx = wd * s[0] / rd, my = wd * s[1] / rd;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(wd * s[2] / rd - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(wd * s[3] / rd - my * my);
    cov[3 * (size_t)c + 2] = (float)(wd * s[4] / rd - mx * my);
}

__global__ __launch_bounds__(256) void k_moments(
    const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ perm,
    const float* __restrict__ pvx, const float* __restrict__ pvy, const uint32_t* __restrict__ offsets,
    const float* __restrict__ rho_p, float2* __restrict__ mean, float* __restrict__ cov,
    MomPartial* __restrict__ head, MomPartial* __restrict__ tail, uint32_t* __restrict__ tail_cell,
    uint8_t* __restrict__ head_ends, const DevScalars* __restrict__ sc, uint32_t nranges)
{
    const int lane = threadIdx.x & 31;
    const uint32_t wr = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (wr >= nranges) return;
    const uint32_t n_in = (uint32_t)sc->n_in;
    const float w_pred = sc->w_pred;
    const uint32_t start = wr * kMomRange;
    if (start >= n_in) {
        if (lane == 0) { tail_cell[wr] = 0xFFFFFFFFu; head_ends[wr] = 1; }
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
        double v[5] = {0, 0, 0, 0, 0};
        if (valid) {
            const uint32_t i = perm[j];
            const double a = (double)pvx[i], bq = (double)pvy[i];
            v[0] = a; v[1] = bq; v[2] = a * a; v[3] = bq * bq; v[4] = a * bq;
        }
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
                // the segment that entered from the previous range ends here: head partial
                MomPartial hp;
#pragma unroll
                for (int q = 0; q < 5; ++q) hp.s[q] = v[q];
                head[wr] = hp;
                head_ends[wr] = 1;
            } else {
                finalize_cell(cell, v, offsets, rho_p, w_pred, mean, cov);
            }
        }
        // carry of lane 31 (or the last valid lane) into the next chunk
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
                head[wr] = p;
                head_ends[wr] = 0;
                tail_cell[wr] = 0xFFFFFFFFu;
            } else {
                tail[wr] = p;
                tail_cell[wr] = carry_cell;
                if (!cont_before) head_ends[wr] = 1;
            }
        } else {
            tail_cell[wr] = 0xFFFFFFFFu;
            if (!cont_before) head_ends[wr] = 1;
        }
    }
}

__global__ void k_moments_fixup(const MomPartial* __restrict__ head, const MomPartial* __restrict__ tail,
                                const uint32_t* __restrict__ tail_cell, const uint8_t* __restrict__ head_ends,
                                const uint32_t* __restrict__ offsets, const float* __restrict__ rho_p,
                                float2* __restrict__ mean, float* __restrict__ cov,
                                const DevScalars* __restrict__ sc, uint32_t nranges)
{
    const uint32_t wr = blockIdx.x * blockDim.x + threadIdx.x;
    if (wr >= nranges) return;
    const uint32_t c = tail_cell[wr];
    if (c == 0xFFFFFFFFu) return;
    double s[5];
    for (int q = 0; q < 5; ++q) s[q] = tail[wr].s[q];
    for (uint32_t r = wr + 1; r < nranges; ++r) {
        for (int q = 0; q < 5; ++q) s[q] += head[r].s[q];
        if (head_ends[r]) break;
    }
    finalize_cell(c, s, offsets, rho_p, sc->w_pred, mean, cov);
}

// ------------------------------------------------------------------------------------------------
// Alg. 5 -- new-born particles (Abar set): slot j -> cell by binary search over the slot starts,
// uniform position inside the cell, v ~ N(0, sigma_B^2 I) (A-16).
// ------------------------------------------------------------------------------------------------
__global__ __launch_bounds__(256) void k_births(const uint32_t* __restrict__ sb, float* __restrict__ bx,
                                                float* __restrict__ by, float* __restrict__ bvx,
                                                float* __restrict__ bvy, const DevScalars* __restrict__ sc,
                                                FilterConst fc, int64_t k)
{
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= fc.nu_b) return;
    if ((uint64_t)j >= sc->s_total) return;
    uint32_t lo = 0, hi = fc.C;                // sb[lo] <= j < sb[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sb[mid] <= j) lo = mid; else hi = mid;
    }
    const uint32_t c = lo;
    const uint32_t col = c % (uint32_t)fc.W, row = c / (uint32_t)fc.W;
    const Philox4 r = draw(fc.seed, j, k, STAGE_BIRTH);
    const float colf = (float)col, rowf = (float)row;
    float x = __fadd_rn(colf, unit24(r.r0));
    float y = __fadd_rn(rowf, unit24(r.r1));
    const float cx1 = __fadd_rn(colf, 1.0f), cy1 = __fadd_rn(rowf, 1.0f);
    if (x >= cx1) x = __int_as_float(__float_as_int(cx1) - 1);   // nextafter(col+1, 0)
    if (y >= cy1) y = __int_as_float(__float_as_int(cy1) - 1);
    float n0, n1;
    box_muller(r.r2, r.r3, n0, n1);
    float vx = __fmul_rn(fc.sigma_b, n0), vy = __fmul_rn(fc.sigma_b, n1);
    if (fc.v_max > 0.0f) {
        vx = fminf(fmaxf(vx, -fc.v_max), fc.v_max);
        vy = fminf(fmaxf(vy, -fc.v_max), fc.v_max);
    }
    bx[j] = x; by[j] = y; bvx[j] = vx; bvy[j] = vy;
}

// ------------------------------------------------------------------------------------------------
// Alg. 7 -- systematic resampling (Eq. 57; A-24): t_i = floor((i 2^32 + U) W / (nu 2^32)); the cell
// with P_c <= t_i < P_{c+1} by binary search over the cell-level CDF, then exact inversion of the
// cell's even split (first R mod n members one unit heavier) -- identical to a particle-level search.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t invert_split(uint64_t o, uint64_t R, uint32_t n)
{
    const uint64_t base = R / n, rem = R % n;
    const uint64_t big = rem * (base + 1);
    if (o < big) return (uint32_t)(o / (base + 1));
    return (uint32_t)(rem + (o - big) / base);
}

__device__ __forceinline__ uint64_t target_of(uint32_t i, uint32_t U, uint64_t W, uint32_t nu)
{
    const u128 X = (((u128)i) << 32) + (u128)U;
    return (uint64_t)((X * (u128)W) / (((u128)nu) << 32));
}

__global__ __launch_bounds__(256) void k_resample(
    const uint64_t* __restrict__ P, const uint32_t* __restrict__ sb, const uint32_t* __restrict__ offsets,
    const uint64_t* __restrict__ Rp, const uint64_t* __restrict__ Rb, const uint32_t* __restrict__ perm,
    const float* __restrict__ px, const float* __restrict__ py, const float* __restrict__ pvx,
    const float* __restrict__ pvy, const float* __restrict__ bx, const float* __restrict__ by,
    const float* __restrict__ bvx, const float* __restrict__ bvy, float* __restrict__ x,
    float* __restrict__ y, float* __restrict__ vx, float* __restrict__ vy, uint32_t* __restrict__ jidx,
    const DevScalars* __restrict__ sc, FilterConst fc)
{
    __shared__ uint32_t s_lo, s_hi;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t W = sc->W;
    if (W == 0) {
        if (i < fc.nu) {
            x[i] = kSentinelPos; y[i] = kSentinelPos; vx[i] = 0.0f; vy[i] = 0.0f;
            if (jidx) jidx[i] = 0xFFFFFFFFu;
        }
        return;
    }
    const uint32_t U = sc->U;
    const uint32_t C = fc.C;
    if (threadIdx.x == 0) {   // narrow the search to the cells of this block's targets
        const uint32_t i0 = blockIdx.x * blockDim.x;
        const uint32_t i1 = min(i0 + blockDim.x, fc.nu) - 1;
        const uint64_t t0 = target_of(i0, U, W, fc.nu), t1 = target_of(i1, U, W, fc.nu);
        uint32_t lo = 0, hi = C;
        while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (P[m] <= t0) lo = m; else hi = m; }
        s_lo = lo;
        uint32_t lo2 = lo; hi = C;
        while (hi - lo2 > 1) { const uint32_t m = (lo2 + hi) >> 1; if (P[m] <= t1) lo2 = m; else hi = m; }
        s_hi = lo2 + 1;
    }
    __syncthreads();
    if (i >= fc.nu) return;
    const uint64_t t = target_of(i, U, W, fc.nu);
    uint32_t lo = s_lo, hi = s_hi;                       // P[lo] <= t < P[hi]
    while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (P[m] <= t) lo = m; else hi = m; }
    const uint32_t c = lo;
    uint64_t o = t - P[c];
    const uint32_t off = offsets[c], n = offsets[c + 1] - off;
    const uint64_t rp = Rp[c];
    float ox, oy, ovx, ovy;
    uint32_t joint;
    if (o < rp) {
        const uint32_t r = invert_split(o, rp, n);
        const uint32_t src = perm[off + r];
        ox = px[src]; oy = py[src]; ovx = pvx[src]; ovy = pvy[src];
        joint = off + sb[c] + r;
    } else {
        o -= rp;
        const uint32_t s0 = sb[c], m = sb[c + 1] - s0;
        const uint32_t r = invert_split(o, Rb[c], m);
        const uint32_t slot = s0 + r;
        ox = bx[slot]; oy = by[slot]; ovx = bvx[slot]; ovy = bvy[slot];
        joint = off + s0 + n + r;
    }
    x[i] = ox; y[i] = oy; vx[i] = ovx; vy[i] = ovy;
    if (jidx) jidx[i] = joint;
}

}  // namespace dog
