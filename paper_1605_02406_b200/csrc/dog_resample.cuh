// dog_resample.cuh -- one fused pass over the joint particle set: velocity moments (Alg. 6,
// Eqs. 81-84), new-born particle initialisation (Alg. 5) and systematic resampling (Alg. 7,
// Eq. 57) to the next state.
//
// Persistent particles are processed tile by tile (k_resample_tiles): the predicted state is read in
// the tile's local sorted order (dog_sort.cuh), so no global permutation pass is needed; births by
// per-cell work items (k_births).
//
// Resampling is member-driven: member r of a cell owns the fixed-point weight range [Q_r, Q_{r+1})
// of the joint CDF (cell prefix P_c plus the even split of the cell's mass, A-23) and writes its
// copies to the outputs i with Q_r <= t_i < Q_{r+1}, t_i = floor((i 2^32 + U) W / (nu 2^32))
// (A-24): i in [F(Q_r), F(Q_{r+1})), F(X) = #{i : t_i < X} = clamp(ceil((X nu 2^32 - U W) / (W 2^32)),
// 0, nu).  This selects exactly what the oracle's binary search over the particle-level CDF selects.
#pragma once
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_rng.cuh"
#include "dog_sort.cuh"

namespace dog {

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
    const u128 num0 = ((u128)X * (u128)r.nu) << 32;
    if (num0 <= r.UW) return 0u;
    const u128 num = num0 - r.UW;
    const u128 E = ((u128)r.W) << 32;
    uint64_t q = (uint64_t)fmax(cy - 1.0, 0.0);
    while ((u128)q * E < num) ++q;                 // smallest q with q W 2^32 >= X nu 2^32 - U W
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

// Last index in [lo, hi) whose value v(idx) <= key, warp-cooperative 32-ary search; assumes
// v(lo) <= key.  Every lane returns the result.
template <typename F>
__device__ __forceinline__ uint32_t warp_last_le(uint32_t lo, uint32_t hi, uint32_t key, F v)
{
    const int lane = threadIdx.x & 31;
    while (hi - lo > 1) {
        const uint32_t span = hi - lo;
        const uint32_t step = (span + 31) / 32;
        const uint32_t p = lo + (uint32_t)lane * step;     // probe lane's position
        const bool ok = p < hi && v(p) <= key;
        const uint32_t m = __ballot_sync(0xffffffffu, ok);   // a prefix of lanes (monotone values)
        const int last = 31 - __clz(m);                      // lane 0 always ok
        lo = lo + (uint32_t)last * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

constexpr int kRtThreads = 256, kRtItems = kSortTile / kRtThreads;   // 16 sorted positions per thread
constexpr int kRtRunCache = 352;                                      // runs whose parameters sit in smem

struct RunParams {
    uint64_t P, bp;
    uint32_t pre, rpm, jbase, key;
};

__device__ __forceinline__ RunParams fetch_run(uint32_t base, uint32_t j, TilePairs tp, CellList L, BlockTotals bt,
                                               uint32_t chunk, const uint32_t* __restrict__ cell2list, uint32_t C)
{
    RunParams q{};
    q.key = tp.key[base + j];
    if (q.key < C) {
        q.pre = tp.pre[base + j];
        const uint32_t li = cell2list[q.key];
        q.P = bt.P0[li / chunk] + L.Pl[li];
        q.bp = L.bp[li];
        q.rpm = L.rp[li];
        q.jbase = L.start[li] + L.sb[li];
    }
    return q;
}

// Persistent particles, one block per sort tile; thread t owns the tile's local sorted positions
// [16t, 16t+16).  Position p of run j (cell c) is member r = pre(j) + (p - first(j)) of cell c: its
// copies go to [F(Q_r), F(Q_{r+1})).  Velocity sums are accumulated per run segment; segments that
// span threads are combined in thread order, and a cell's runs over the tiles in tile order by the
// last run to finish (deterministic).
__global__ __launch_bounds__(kRtThreads, 4) void k_resample_tiles(
    const uint16_t* __restrict__ lperm, TilePairs tp, Pred pr, CellList L, BlockTotals bt, uint32_t chunk,
    const uint32_t* __restrict__ cell2list, const uint32_t* __restrict__ plist, NextState out,
    uint32_t* __restrict__ perm_dbg, float2* __restrict__ mean, float* __restrict__ cov,
    MomPartial* __restrict__ ppart, const DevScalars* __restrict__ sc, FilterConst fc)
{
    __shared__ __align__(16) uint16_t s_lp[kSortTile];
    __shared__ __align__(16) uint16_t s_first[kSortTile + 8];
    __shared__ MomPartial s_pa[kRtThreads], s_pb[kRtThreads];
    __shared__ RunParams s_run[kRtRunCache];
    const int tid = threadIdx.x;
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    const RsConst rc = make_rsconst(sc, fc.nu);
    if (rc.W == 0) {   // empty world (A-26): every next particle goes to the sentinel
        for (uint32_t i = blockIdx.x * blockDim.x + tid; i < fc.nu; i += gridDim.x * blockDim.x) {
            out.x[i] = kSentinelPos; out.y[i] = kSentinelPos; out.vx[i] = 0.0f; out.vy[i] = 0.0f;
            if (out.jidx) out.jidx[i] = 0xFFFFFFFFu;
        }
    }
    const uint32_t n = fc.nu > base ? min((uint32_t)kSortTile, fc.nu - base) : 0u;
    if (n == 0) return;
    const uint32_t nd = tp.nd[t];
    const float w_pred = sc->w_pred;
    const uint32_t p0 = tid * kRtItems;
    {   // one round trip: 16 local indices and 16 run starts per thread (32-byte vector loads)
        const uint4* lp4 = reinterpret_cast<const uint4*>(lperm + base + p0);
        const uint4* fi4 = reinterpret_cast<const uint4*>(tp.first + base + p0);
        uint4 a = make_uint4(0, 0, 0, 0), b = a, c = a, d = a;
        if (p0 < n) { a = lp4[0]; b = lp4[1]; }
        if (p0 < nd) { c = fi4[0]; d = fi4[1]; }
        if (p0 < n) { reinterpret_cast<uint4*>(s_lp + p0)[0] = a; reinterpret_cast<uint4*>(s_lp + p0)[1] = b; }
        if (p0 < nd) { reinterpret_cast<uint4*>(s_first + p0)[0] = c; reinterpret_cast<uint4*>(s_first + p0)[1] = d; }
    }
    for (uint32_t r = tid; r < nd && r < (uint32_t)kRtRunCache; r += kRtThreads)
        s_run[r] = fetch_run(base, r, tp, L, bt, chunk, cell2list, fc.C);
    __syncthreads();
    if (tid == 0) s_first[nd] = (uint16_t)n;
    __syncthreads();

    if (p0 < n) {
        uint32_t lo = 0, hi = nd;                           // run containing p0
        while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (s_first[m] <= p0) lo = m; else hi = m; }
        uint32_t j = lo, first = s_first[j], end = s_first[j + 1];
        RunParams q = j < (uint32_t)kRtRunCache ? s_run[j] : fetch_run(base, j, tp, L, bt, chunk, cell2list, fc.C);
        double acc[5] = {0, 0, 0, 0, 0};
        bool first_seg = true;
        uint32_t F_next = 0xFFFFFFFFu;                      // F(Q_{r+1}) of the previous position, same run
        const uint32_t pend = min(p0 + (uint32_t)kRtItems, n);
        auto flush = [&]() {
            MomPartial mp;
#pragma unroll
            for (int i = 0; i < 5; ++i) { mp.s[i] = acc[i]; acc[i] = 0.0; }
            if (q.key < fc.C) {
                if (first >= p0 && end <= pend) ppart[base + j] = mp;    // run inside this thread
                else if (first_seg) s_pa[tid] = mp;
                else s_pb[tid] = mp;
            }
            first_seg = false;
        };
#pragma unroll 1
        for (uint32_t b0 = p0; b0 < pend; b0 += 8) {
            float X[8], Y[8], VX[8], VY[8];
            uint32_t src[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) src[u] = base + s_lp[min(b0 + u, pend - 1)];
#pragma unroll
            for (int u = 0; u < 8; ++u) { X[u] = pr.x[src[u]]; Y[u] = pr.y[src[u]]; VX[u] = pr.vx[src[u]]; VY[u] = pr.vy[src[u]]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t p = b0 + u;
                if (p >= pend) break;
                if (p >= end) {                             // next run
                    flush();
                    ++j; first = end; end = s_first[j + 1];
                    q = j < (uint32_t)kRtRunCache ? s_run[j] : fetch_run(base, j, tp, L, bt, chunk, cell2list, fc.C);
                    F_next = 0xFFFFFFFFu;
                }
                if (q.key >= fc.C) continue;
                const double a = (double)VX[u], bq = (double)VY[u];
                acc[0] += a; acc[1] += bq; acc[2] += a * a; acc[3] += bq * bq; acc[4] += a * bq;
                const uint32_t mr = q.pre + (p - first);    // member rank within the cell
                if (perm_dbg) perm_dbg[q.jbase - L.sb[cell2list[q.key]] + mr] = src[u];
                if (rc.W) {
                    const uint64_t Q0 = q.P + (uint64_t)mr * q.bp + min(mr, q.rpm);
                    const uint32_t F0 = F_next != 0xFFFFFFFFu ? F_next : fcount(Q0, rc);
                    const uint32_t F1 = fcount(Q0 + q.bp + (mr < q.rpm ? 1u : 0u), rc);
                    F_next = F1;
                    for (uint32_t o = F0; o < F1; ++o) {
                        out.x[o] = X[u]; out.y[o] = Y[u]; out.vx[o] = VX[u]; out.vy[o] = VY[u];
                        if (out.jidx) out.jidx[o] = q.jbase + mr;
                    }
                }
            }
        }
        flush();
    }
    __syncthreads();
    // runs spanning several threads: combine the segments in thread order
    for (uint32_t r = tid; r < nd; r += kRtThreads) {
        const uint32_t f = s_first[r], e = s_first[r + 1];
        if (tp.key[base + r] >= fc.C) continue;
        const uint32_t tf = f / kRtItems, tl = (e - 1) / kRtItems;
        if (tf == tl) continue;                             // written directly
        MomPartial mp = (f > tf * kRtItems) ? s_pb[tf] : s_pa[tf];
        for (uint32_t u = tf + 1; u <= tl; ++u)
#pragma unroll
            for (int i = 0; i < 5; ++i) mp.s[i] += s_pa[u].s[i];
        ppart[base + r] = mp;
    }
    __syncthreads();
    // cell completion: the last of a cell's runs to finish combines them in tile order (deterministic)
    for (uint32_t r = tid; r < nd; r += kRtThreads) {
        const uint32_t key = tp.key[base + r];
        if (key >= fc.C) continue;
        const uint32_t li = cell2list[key];
        const uint32_t m = L.np[li];
        if (m == 1) {
            finalize_cell(key, ppart[base + r].s, L.n[li], L.rho_p[li], w_pred, mean, cov);
            continue;
        }
        __threadfence();
        if (atomicAdd(&L.pdone[li], 1u) != m - 1) continue;
        __threadfence();
        const uint32_t* pl = plist + bt.ps0[li / chunk] + L.ps[li];
        double sum[5] = {0, 0, 0, 0, 0};
        for (uint32_t qq = 0; qq < m; ++qq) {
            const double* ps = ppart[pl[qq]].s;
#pragma unroll
            for (int i = 0; i < 5; ++i) sum[i] += __ldcg(ps + i);
        }
        finalize_cell(key, sum, L.n[li], L.rho_p[li], w_pred, mean, cov);
    }
}

// New-born particles (Alg. 5): work items of <= 256 birth slots of one cell; each warp takes a
// contiguous range of items.  State from the slot's Philox draw; copies as for persistent members.
__global__ __launch_bounds__(256) void k_births(CellList L, BlockTotals bt, uint32_t nblk, uint32_t chunk,
                                                NextState out, BirthDebug bdbg, const DevScalars* __restrict__ sc,
                                                FilterConst fc, int64_t k)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const RsConst rc = make_rsconst(sc, fc.nu);
    const uint32_t n_items = sc->n_items;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    const uint32_t per = (n_items + nwarps - 1) / nwarps;
    uint32_t q = gw * per;
    const uint32_t q_end = min(q + per, n_items);
    if (q >= q_end) return;
    uint32_t b = warp_last_le(0u, nblk, q, [&](uint32_t i) { return bt.item0[i]; });
    uint32_t lbase = b * chunk;
    uint32_t li = warp_last_le(lbase, lbase + bt.cnt[b], q - bt.item0[b], [&](uint32_t i) { return L.it[i]; });
    uint32_t sub = q - bt.item0[b] - L.it[li];
    while (true) {
        const uint32_t c = L.c[li], n = L.n[li], start = L.start[li], nb = L.nb[li];
        const uint64_t P = bt.P0[b] + L.Pl[li];
        const uint32_t r0 = sub * kItem, m = min(kItem, nb - r0);
        const uint64_t bb = L.bb[li];
        const uint32_t rbm = L.rb[li], sb = L.sb[li];
        const uint64_t PB = P + L.Rp[li];
        const uint32_t jbase = start + sb + n;
        const uint32_t col = c % (uint32_t)fc.W, row = c / (uint32_t)fc.W;
        const float colf = (float)col, rowf = (float)row;
        const float cx1 = __fadd_rn(colf, 1.0f), cy1 = __fadd_rn(rowf, 1.0f);
        for (uint32_t t = 0; t < m; t += 32) {
            const bool valid = t + lane < m;
            const uint32_t r = r0 + t + lane;
            const uint32_t s = sb + r;
            const Philox4 d = draw(fc.seed, s, k, STAGE_BIRTH);
            float bx = __fadd_rn(colf, unit24(d.r0));
            float by = __fadd_rn(rowf, unit24(d.r1));
            if (bx >= cx1) bx = __int_as_float(__float_as_int(cx1) - 1);    // nextafter(col+1, 0) (A-16)
            if (by >= cy1) by = __int_as_float(__float_as_int(cy1) - 1);
            float n0, n1;
            box_muller(d.r2, d.r3, n0, n1);
            float bvx = __fmul_rn(fc.sigma_b, n0), bvy = __fmul_rn(fc.sigma_b, n1);
            if (fc.v_max > 0.0f) {
                bvx = fminf(fmaxf(bvx, -fc.v_max), fc.v_max);
                bvy = fminf(fmaxf(bvy, -fc.v_max), fc.v_max);
            }
            if (valid && bdbg.x) { bdbg.x[s] = bx; bdbg.y[s] = by; bdbg.vx[s] = bvx; bdbg.vy[s] = bvy; }
            if (rc.W) {
                const uint64_t Q0 = PB + (uint64_t)r * bb + min(r, rbm);
                const uint32_t F0 = valid ? fcount(Q0, rc) : 0u;
                uint32_t F1 = __shfl_down_sync(0xffffffffu, F0, 1);
                if (valid && (lane == 31 || t + lane + 1 == m)) F1 = fcount(Q0 + bb + (r < rbm ? 1u : 0u), rc);
                if (valid) {
                    for (uint32_t o = F0; o < F1; ++o) {
                        out.x[o] = bx; out.y[o] = by; out.vx[o] = bvx; out.vy[o] = bvy;
                        if (out.jidx) out.jidx[o] = jbase + r;
                    }
                }
            }
        }
        if (++q >= q_end) break;
        if (++sub < (nb + kItem - 1) / kItem) continue;
        sub = 0;
        const uint32_t chunk_end = b + 1 < nblk ? bt.item0[b + 1] : n_items;
        if (q >= chunk_end) b = warp_last_le(b, nblk, q, [&](uint32_t i) { return bt.item0[i]; });
        const uint32_t lo = q >= chunk_end ? b * chunk : li + 1;
        lbase = b * chunk;
        li = warp_last_le(lo, lbase + bt.cnt[b], q - bt.item0[b], [&](uint32_t i) { return L.it[i]; });
        sub = q - bt.item0[b] - L.it[li];
    }
}

}  // namespace dog
