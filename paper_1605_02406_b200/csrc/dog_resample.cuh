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
#include <cstddef>
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_rng.cuh"
#include "dog_sort.cuh"

namespace dog {

struct MomPartial { double s[5]; };

// Moments of cell c from its velocity sums (Eqs. 81-84 with the uniform weight w' = rho_p / S w_pred).
__device__ __forceinline__ void finalize_cell(uint32_t c, double s0, double s1, double s2, double s3, double s4,
                                              uint32_t n, float rp, float w_pred, float2* __restrict__ mean,
                                              float* __restrict__ cov)
{
    const float S = __double2float_rn(__dmul_rn((double)n, (double)w_pred));
    if (!(rp > 0.0f) || !(S > 0.0f)) return;
    const float w = __fmul_rn(__fdiv_rn(rp, S), w_pred);       // Eq. 71 with p_A = 0, Eq. 73
    const double wd = (double)w, rd = (double)rp;
    const double mx = wd * s0 / rd, my = wd * s1 / rd;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(wd * s2 / rd - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(wd * s3 / rd - my * my);
    cov[3 * (size_t)c + 2] = (float)(wd * s4 / rd - mx * my);
}

// Moments of a Doppler cell (NEXT-1, A-35): sums weighted by the members' fixed-point weights q_j,
// normalised by their total R_p.
__device__ __forceinline__ void finalize_cell_dop(uint32_t c, double s0, double s1, double s2, double s3, double s4,
                                                  uint64_t Rp, float2* __restrict__ mean, float* __restrict__ cov)
{
    if (Rp == 0) {
        mean[c] = make_float2(0.0f, 0.0f);
        cov[3 * (size_t)c] = 0.0f; cov[3 * (size_t)c + 1] = 0.0f; cov[3 * (size_t)c + 2] = 0.0f;
        return;
    }
    const double rd = (double)Rp;
    const double mx = s0 / rd, my = s1 / rd;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(s2 / rd - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(s3 / rd - my * my);
    cov[3 * (size_t)c + 2] = (float)(s4 / rd - mx * my);
}

struct NextState { float4* s; uint32_t* jidx; };   // (x, y, vx, vy) per particle; joint index (debug)
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

// Warp-cooperative write of the copies of 32 consecutive members (lanes): member l owns outputs
// [F0_l, F1_l), consecutive members own consecutive ranges, so the warp's outputs are one contiguous
// range [F0_0, F1_last) written 32 at a time; the owner of output o is found by a 5-step shuffle
// search.  Balanced and coalesced whatever the copy counts (a member can own hundreds of outputs).
__device__ __forceinline__ void write_copies(bool valid, uint32_t F0, uint32_t F1, float X, float Y, float VX,
                                             float VY, uint32_t J, NextState& out)
{
    const int lane = threadIdx.x & 31;
    const uint32_t vm = __ballot_sync(0xffffffffu, valid);
    if (!vm) return;
    const int lastv = 31 - __clz(vm);
    const uint32_t lo = __shfl_sync(0xffffffffu, F0, __ffs(vm) - 1);
    const uint32_t hi = __shfl_sync(0xffffffffu, F1, lastv);
    const uint32_t f0 = valid ? F0 : hi;                    // invalid lanes own nothing
    for (uint32_t o0 = lo; o0 < hi; o0 += 32) {
        const uint32_t o = o0 + lane;
        int own = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const int cand = own + step;
            const uint32_t f = __shfl_sync(0xffffffffu, f0, cand);
            if (f <= o) own = cand;
        }
        const float x = __shfl_sync(0xffffffffu, X, own), y = __shfl_sync(0xffffffffu, Y, own);
        const float vx = __shfl_sync(0xffffffffu, VX, own), vy = __shfl_sync(0xffffffffu, VY, own);
        const uint32_t jj = __shfl_sync(0xffffffffu, J, own);
        if (o < hi) {
            out.s[o] = make_float4(x, y, vx, vy);
            if (out.jidx) out.jidx[o] = jj;
        }
    }
}

#ifndef RT_THREADS
#define RT_THREADS 256
#endif
#ifndef RT_MINB
#define RT_MINB (1024 / RT_THREADS)
#endif
constexpr int kRtThreads = RT_THREADS, kRtItems = kSortTile / kRtThreads;   // sorted positions per thread
static_assert(kRtItems % 8 == 0, "phase B works in batches of 8 positions");
constexpr int kRtRunCache = 96;                                       // runs whose RunF sits in smem (rest: global)
constexpr uint32_t kRtShortSpan = 8;                                  // phase R: longer runs combined by a warp
constexpr int kRtWin = 8192;                                          // compact outputs per phase-C window
constexpr int kRtWinItems = kRtWin / kRtThreads;                      // 32 window entries per thread

// Per run, everything the owner marks need: F(Q_r) of member r = pre + k (k = position - first) is
// ceil(y) with y = y0 + r d1 for r <= rpm and yR + (r - rpm) d2 beyond (Q is linear in r on both
// pieces, steps bp + 1 and bp); D = F(Q_pre) - the run's offset in the tile's compact output space.
struct RunF {
    double y0, d1;          // the second piece (members beyond rpm) is derived: yR = y0 + rpm d1, d2 = d1 - nu/W
    uint32_t pre, rpm, D, pad;
};
static_assert(sizeof(RunF) == 32, "RunF: two per 64-byte line");

struct RtSmem {   // dynamic shared memory of k_resample_tiles (~47 KB: three blocks per SM with a large L1)
    uint16_t lp[kSortTile];            // local sorted position -> local index
    uint16_t first[kSortTile + 8];     // run starts (first[nd] = n)
    uint16_t runof[kSortTile];         // sorted position -> run
    alignas(16) RunF rf[kRtRunCache];
    union alignas(16) {
        struct { MomPartial pa[kRtThreads], pb[kRtThreads]; } m;   // phase B -> phase R
        uint16_t osrc[kRtWin];         // phase C: compact output -> owner position + 1
    } u;
    uint32_t scan[kRtThreads / 32 + 1];
    uint32_t sentinel_run;             // index of the run outside the grid, or 0xFFFFFFFF
    uint32_t nlong;                    // runs spanning more than kRtShortSpan threads (phase R)
    uint16_t longr[32];
    uint32_t slow;                     // an estimate was too close to an integer: exact marks needed
};
constexpr size_t kRtSmemBytes = sizeof(RtSmem);
static_assert(offsetof(RtSmem, u) % 16 == 0 && offsetof(RtSmem, runof) % 16 == 0, "vector smem access");

// ceil(y) clamped to [0, nu] when y is further than `margin` from an integer; otherwise *amb is set (the
// caller redoes the work with exact products).  The per-run linear estimates are within ~nu 2^-50 of
// the exact value, so margin = max(2^-22, nu 2^-48) keeps every accepted ceil exact.
__device__ __forceinline__ double fast_ceil_margin(uint32_t nu) { return fmax(0x1p-22, (double)nu * 0x1p-48); }
__device__ __forceinline__ uint32_t fast_ceil(double y, uint32_t nu, double margin, bool& amb)
{
    if (y <= -0.5) return 0u;
    if (y >= (double)nu) return nu;
    const double cy = ceil(y);
    const double d = cy - y;
    amb |= !(d > margin && d < 1.0 - margin);
    return (uint32_t)cy;
}

// Block-wide exclusive max-scan of one value per thread (values >= 0).
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* s_warp)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = max(inc, o);
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < warp; ++w) pre = max(pre, s_warp[w]);
    const uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    __syncthreads();
    return max(pre, lane ? ex : 0u);
}

// Q of member mr of a run's cell: P + mr bp + min(mr, rpm) (even split of the cell's R_p, A-23).
__device__ __forceinline__ uint64_t member_Q(const RunInfo& q, uint32_t mr)
{
    return q.P + (uint64_t)mr * q.bp + min(mr, q.rpm);
}

// Persistent particles, one block per sort tile (4096 particles in input order; lperm gives their
// stable cell order).
//   phase B (thread t owns sorted positions [16t, 16t+16)): run of every position, batched gathers of
//     the predicted velocities, velocity sums per run segment (runs inside a thread -> ppart directly).
//   phase R (thread per run): run segments spanning threads combined in thread order (deterministic)
//     -> ppart; the run's output range [F(Q_first), F(Q_end)) and its offset in the tile's compact
//     output space (the runs' ranges concatenated).
//   phase C, per window of 4096 compact outputs: lanes take consecutive positions, compute F(Q_r) of
//     their member (the next member's from the neighbour lane) and mark the member's first output; a
//     block max-scan spreads the owner over its outputs; threads write consecutive outputs (coalesced,
//     balanced whatever the copy counts).
template <bool kDbg>
__global__ __launch_bounds__(kRtThreads, RT_MINB) void k_resample_tiles(
    const uint16_t* __restrict__ lperm, TilePairs tp, const float4* __restrict__ pred, CellList L, NextState out,
    uint32_t* __restrict__ perm_dbg, MomPartial* __restrict__ ppart, RunF* __restrict__ rf_g,
    const DevScalars* __restrict__ sc, FilterConst fc, int par, const uint8_t* __restrict__ tskip)
{
    PDL_ENTER();
    const double fmargin = fast_ceil_margin(fc.nu);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    RtSmem& S = *reinterpret_cast<RtSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint32_t t = blockIdx.x, base = t * kSortTile;     // this tile's slot in the per-tile arrays
    const RsConst rc = make_rsconst(sc, fc.nu);
    const uint32_t n_lo = sc->n_lo, n_loc = n_lo + sc->n_own[par] + sc->n_hi;
    const uint32_t pbase = fc.lo_cap - n_lo + base;                // its first particle
    // next-cycle own particles start at lo_cap: global output o -> slot lo_cap + o - F(P'_shard)
    out.s += fc.lo_cap - sc->o_base[par ^ 1];
    if (rc.W == 0 && fc.world == 1) {   // empty world (A-26): every next particle goes to the sentinel
        for (uint32_t i = blockIdx.x * blockDim.x + tid; i < fc.nu; i += gridDim.x * blockDim.x) {
            out.s[i] = make_float4(kSentinelPos, kSentinelPos, 0.0f, 0.0f);
            if (kDbg) out.jidx[i] = 0xFFFFFFFFu;
        }
    }
    const uint32_t n = n_loc > base ? min((uint32_t)kSortTile, n_loc - base) : 0u;
    if (n == 0) return;
    if (tskip && tskip[t]) return;                                 // a Doppler tile (k_resample_dopp)
    const uint32_t nd = tp.nd[t];
    const uint32_t p0 = tid * kRtItems;
    const RunInfo* __restrict__ runs = tp.run + base;
    PHASE_BEGIN();
    // ---- phase A: local permutation, run starts
    const float2* __restrict__ pv = reinterpret_cast<const float2*>(pred);   // (x, y), (vx, vy) halves
    {
        uint4 a = make_uint4(0, 0, 0, 0), b = a, c = a, d = a;
#pragma unroll
        for (int h = 0; h < kRtItems / 8; ++h) {
            if (p0 < n) { a = reinterpret_cast<const uint4*>(lperm + base + p0)[h]; reinterpret_cast<uint4*>(S.lp + p0)[h] = a; }
            if (p0 < nd) { c = reinterpret_cast<const uint4*>(tp.first + base + p0)[h]; reinterpret_cast<uint4*>(S.first + p0)[h] = c; }
        }
        (void)b; (void)d;
        if (tid == 0) { S.slow = 0u; S.nlong = 0u; }
        if (tid == 0) S.sentinel_run = tp.key[base + nd - 1] >= fc.C ? nd - 1 : 0xFFFFFFFFu;
    }
    __syncthreads();
    if (tid == 0) S.first[nd] = (uint16_t)n;
    __syncthreads();
    const uint32_t srun = S.sentinel_run;
    auto runf = [&](uint32_t j) -> const RunF& { return j < (uint32_t)kRtRunCache ? S.rf[j] : rf_g[base + j]; };

    PHASE_MARK(0);
    // ---- phase B: run of every position, velocity sums per run segment
    if (p0 < n) {
        uint32_t lo = 0, hi = nd;                           // run containing p0
        while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (S.first[m] <= p0) lo = m; else hi = m; }
        uint32_t j = lo, first = S.first[j], end = S.first[j + 1];
        double acc[5] = {0, 0, 0, 0, 0};
        bool first_seg = true;
        auto flush = [&]() {
            MomPartial mp;
#pragma unroll
            for (int i = 0; i < 5; ++i) { mp.s[i] = acc[i]; acc[i] = 0.0; }
            if (j != srun) {
                if (first >= p0 && end <= p0 + kRtItems) ppart[base + j] = mp;    // run inside this thread
                else if (first_seg) S.u.m.pa[tid] = mp;
                else S.u.m.pb[tid] = mp;
            }
            first_seg = false;
        };
#pragma unroll 1
        for (int h = 0; h < kRtItems / 8; ++h) {            // batches of 8 positions
            uint32_t src[8], rpk[4];
            {
                const uint4 a = reinterpret_cast<const uint4*>(S.lp + p0)[h];
                const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) { src[2 * u] = pbase + (w[u] & 0xFFFFu); src[2 * u + 1] = pbase + (w[u] >> 16); }
            }
            float2 V[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                V[u] = (p0 + 8 * h + u < n) ? pv[2 * (size_t)src[u] + 1] : make_float2(0.0f, 0.0f);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t p = p0 + 8 * h + u;
                if (p < n) {
                    if (p >= end) {                         // next run
                        flush();
                        ++j; first = end; end = S.first[j + 1];
                    }
                    if (j != srun) {
                        const double a = (double)V[u].x, bq = (double)V[u].y;
                        acc[0] += a; acc[1] += bq; acc[2] += a * a; acc[3] += bq * bq; acc[4] += a * bq;
                        if (kDbg) {
                            const RunInfo q = runs[j];
                            perm_dbg[q.jbase - L.sb[q.li] + q.pre + (p - first)] = src[u];
                        }
                    }
                }
                if (u & 1) rpk[u >> 1] |= j << 16; else rpk[u >> 1] = j;
            }
            reinterpret_cast<uint4*>(S.runof + p0)[h] = make_uint4(rpk[0], rpk[1], rpk[2], rpk[3]);
        }
        flush();
    }
    __syncthreads();
    PHASE_MARK(1);
    // ---- phase R: spanning run segments -> ppart; output range and compact offset of every run
    uint32_t carry = 0;
    for (uint32_t r0 = 0; r0 < nd; r0 += kRtThreads) {
        const uint32_t r = r0 + tid;
        const bool live = r < nd && r != srun;
        uint32_t Flo = 0, c = 0;
        RunF x{};
        if (live) {
            const uint32_t f = S.first[r], e = S.first[r + 1];
            const uint32_t tf = f / kRtItems, tl = (e - 1) / kRtItems;
            bool by_warp = false;
            if (tl - tf > kRtShortSpan) {                   // long run: combined by a warp after this loop
                const uint32_t k = atomicAdd(&S.nlong, 1u);
                if (k < 32u) { S.longr[k] = (uint16_t)r; by_warp = true; }
            }
            if (tf != tl && !by_warp) {                     // segments over threads tf..tl, in thread order
                const MomPartial& m0 = (f > tf * kRtItems) ? S.u.m.pb[tf] : S.u.m.pa[tf];
                double s5[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) s5[i] = m0.s[i];
                for (uint32_t u = tf + 1; u <= tl; ++u)
#pragma unroll
                    for (int i = 0; i < 5; ++i) s5[i] += S.u.m.pa[u].s[i];
                MomPartial mp;
#pragma unroll
                for (int i = 0; i < 5; ++i) mp.s[i] = s5[i];
                ppart[base + r] = mp;
            }
            if (rc.W) {   // F at the run's ends from the same linear estimate phase C uses (exact unless
                          // ambiguous, then the exact 128-bit count)
                const RunInfo q = runs[r];
                x.y0 = __fma_rn((double)q.P, rc.nu_over_W, -rc.U_frac);
                x.d1 = __dmul_rn((double)(q.bp + 1u), rc.nu_over_W);
                x.pre = q.pre; x.rpm = q.rpm;
                x.pad = 0u;
                const double yR = __fma_rn((double)x.rpm, x.d1, x.y0), d2 = x.d1 - rc.nu_over_W;
                auto yof = [&](uint32_t mr) {
                    return mr <= x.rpm ? __fma_rn((double)mr, x.d1, x.y0) : __fma_rn((double)(mr - x.rpm), d2, yR);
                };
                bool amb = false;
                Flo = fast_ceil(yof(q.pre), rc.nu, fmargin, amb);
                uint32_t Fhi = fast_ceil(yof(q.pre + (e - f)), rc.nu, fmargin, amb);
                if (amb) {
                    Flo = fcount(member_Q(q, q.pre), rc);
                    Fhi = fcount(member_Q(q, q.pre + (e - f)), rc);
                }
                c = Fhi - Flo;
            }
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan<uint32_t, kRtThreads / 32>(c, S.scan, tot);
        if (live && rc.W) {
            x.D = Flo - (carry + ex);
            if (r < (uint32_t)kRtRunCache) S.rf[r] = x; else rf_g[base + r] = x;
        }
        carry += tot;
    }
    __syncthreads();
    {   // long runs: their thread partials summed by one warp each (fixed lane tree: deterministic)
        const uint32_t nlong = min(S.nlong, 32u);
        if (nlong > 0u) {
            const int warp = tid >> 5, lane = tid & 31;
            for (uint32_t k = warp; k < nlong; k += kRtThreads / 32) {
                const uint32_t r = S.longr[k];
                const uint32_t f = S.first[r], e = S.first[r + 1];
                const uint32_t tf = f / kRtItems, tl = (e - 1) / kRtItems;
                double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (uint32_t u = tf + 1 + lane; u <= tl; u += 32)
#pragma unroll
                    for (int i = 0; i < 5; ++i) s5[i] += S.u.m.pa[u].s[i];
#pragma unroll
                for (int d = 16; d; d >>= 1)
#pragma unroll
                    for (int i = 0; i < 5; ++i) s5[i] += __shfl_xor_sync(0xffffffffu, s5[i], d);
                if (lane == 0) {
                    const MomPartial& m0 = (f > tf * kRtItems) ? S.u.m.pb[tf] : S.u.m.pa[tf];
                    MomPartial mp;
#pragma unroll
                    for (int i = 0; i < 5; ++i) mp.s[i] = m0.s[i] + s5[i];
                    ppart[base + r] = mp;
                }
            }
            __syncthreads();                                // phase C reuses the partials' memory
        }
    }
    const uint32_t Ot = carry;
    PHASE_MARK(2);
    // ---- phase C: windows of the compact output space
    uint16_t* os = S.u.osrc;
    const uint32_t q0 = tid * kRtWinItems;                  // this thread's window entries in the max-scan
    for (uint32_t w0 = 0; w0 < Ot; w0 += kRtWin) {
#pragma unroll
        for (int i = 0; i < kRtWinItems / 8; ++i) reinterpret_cast<uint4*>(os + q0)[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        bool amb = false;
        if (p0 < n) {   // members with copies mark their first output in the window: thread-contiguous
                        // positions, the run's F parameters held in registers, F(Q_{r+1}) reused as the next
                        // member's F(Q_r)
            const uint32_t pend = min(p0 + (uint32_t)kRtItems, n);
            uint32_t j = S.runof[p0], end = S.first[j + 1];
            RunF x{};
            double yR = 0.0, d2 = 0.0;                      // the run's second piece (see RunF)
            uint32_t xfirst = S.first[j];
            auto load = [&]() { x = runf(j); yR = __fma_rn((double)x.rpm, x.d1, x.y0); d2 = x.d1 - rc.nu_over_W; };
            if (j != srun) load();
            bool have = false;
            uint32_t Fc = 0;
            for (uint32_t p = p0; p < pend; ++p) {
                if (p >= end) {
                    j = S.runof[p]; xfirst = end; end = S.first[j + 1];
                    if (j != srun) load();
                    have = false;
                }
                if (j == srun) continue;
                const uint32_t mr = x.pre + (p - xfirst);
                uint32_t F0 = Fc;
                if (!have) {
                    const double y = mr <= x.rpm ? __fma_rn((double)mr, x.d1, x.y0) : __fma_rn((double)(mr - x.rpm), d2, yR);
                    F0 = fast_ceil(y, rc.nu, fmargin, amb);
                }
                const double y1 = mr < x.rpm ? __fma_rn((double)(mr + 1u), x.d1, x.y0) : __fma_rn((double)(mr + 1u - x.rpm), d2, yR);
                const uint32_t F1 = fast_ceil(y1, rc.nu, fmargin, amb);
                Fc = F1;
                have = true;
                const uint32_t C0 = F0 - x.D, C1 = F1 - x.D;
                if (C1 > C0 && C1 > w0 && C0 < w0 + kRtWin) os[max(C0, w0) - w0] = (uint16_t)(p + 1u);
            }
        }
        if (amb) S.slow = 1u;
        __syncthreads();
#ifdef DOG_TIMING
        if (S.slow && tid == 0) atomicAdd(&g_phase_ns[20], 1ull);
        if (tid == 0) atomicAdd(&g_phase_ns[21], 1ull);
#endif
        if (S.slow) {   // rare: some estimate was ambiguous -- redo the marks with exact products
#pragma unroll
            for (int i = 0; i < kRtWinItems / 8; ++i) reinterpret_cast<uint4*>(os + q0)[i] = make_uint4(0, 0, 0, 0);
            __syncthreads();
            for (int it = 0; it < kRtItems; ++it) {
                const uint32_t p = it * kRtThreads + tid;
                if (p >= n) break;
                const uint32_t j = S.runof[p];
                if (j == srun) continue;
                const RunInfo q = runs[j];
                const RunF& x = runf(j);
                const uint32_t mr = q.pre + (p - S.first[j]);
                const uint64_t Q0 = member_Q(q, mr);
                const uint32_t C0 = fcount(Q0, rc) - x.D;
                const uint32_t C1 = fcount(Q0 + q.bp + (mr < q.rpm ? 1u : 0u), rc) - x.D;
                if (C1 > C0 && C1 > w0 && C0 < w0 + kRtWin) os[max(C0, w0) - w0] = (uint16_t)(p + 1u);
            }
            __syncthreads();
        }
        PHASE_MARK(3);
        {   // inclusive max-scan over the window: thread-contiguous 32 entries (u16 pairs)
            uint32_t v[kRtWinItems / 2];
#pragma unroll
            for (int i = 0; i < kRtWinItems / 8; ++i) {
                const uint4 x = reinterpret_cast<const uint4*>(os + q0)[i];
                v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
            }
            uint32_t run = 0;
#pragma unroll
            for (int i = 0; i < kRtWinItems / 2; ++i) {
                const uint32_t lo = max(v[i] & 0xFFFFu, run), hi = max(v[i] >> 16, lo);
                v[i] = lo | (hi << 16);
                run = hi;
            }
            const uint32_t pre = block_excl_max(run, S.scan);
            const uint32_t pre2 = pre | (pre << 16);
#pragma unroll
            for (int i = 0; i < kRtWinItems / 8; ++i)
                reinterpret_cast<uint4*>(os + q0)[i] = make_uint4(__vmaxu2(v[4 * i], pre2), __vmaxu2(v[4 * i + 1], pre2),
                                                                  __vmaxu2(v[4 * i + 2], pre2), __vmaxu2(v[4 * i + 3], pre2));
        }
        __syncthreads();
        PHASE_MARK(4);
        const uint32_t wn = min((uint32_t)kRtWin, Ot - w0);
#pragma unroll 1
        for (uint32_t i0 = 0; i0 < wn; i0 += 4 * kRtThreads) {
            uint32_t o[4], src[4], J[4];
            bool ok[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint32_t i = i0 + h * kRtThreads + tid;
                ok[h] = i < wn;
                const uint32_t p = (uint32_t)os[ok[h] ? i : 0u] - 1u;
                const uint32_t j = S.runof[p];
                o[h] = w0 + i + runf(j).D;
                src[h] = pbase + S.lp[p];
                J[h] = 0;
                if (kDbg) { const RunInfo q = runs[j]; J[h] = q.jbase + q.pre + (p - S.first[j]); }
            }
            float4 X[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) X[h] = pred[src[h]];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (!ok[h]) continue;
                DOG_ASSERT(o[h] < fc.nu);
                out.s[o[h]] = X[h];
                if (kDbg) out.jidx[o[h]] = J[h];
            }
        }
        __syncthreads();
        PHASE_MARK(5);
    }
}

// Velocity moments per cell (Eqs. 81-84): the cell's run sums combined in tile order (k_pair_sort left
// the run list in that order) in a fixed summation order.  Groups of 8 lanes take one cell each.
constexpr int kMoGroup = 8;
constexpr int kMoSmall = 4;   // kBatch (exact filter): cells with <= 4 runs summed by one lane each

template <bool kBatch>
__global__ __launch_bounds__(256) void k_moments(CellList L, const uint32_t* __restrict__ plist,
                                                 const MomPartial* __restrict__ ppart, float2* __restrict__ mean,
                                                 float* __restrict__ cov, const DevScalars* __restrict__ sc,
                                                 const uint64_t* __restrict__ GSd)
{
    PDL_ENTER();
    const int lane = threadIdx.x & 31, gl = lane & (kMoGroup - 1);
    const uint32_t gmask = 0xFFu << (lane & ~(kMoGroup - 1));
    const uint32_t Lc = sc->Lc;
    const float w_pred = sc->w_pred;
    auto finalize = [&](uint32_t li, const double (&s5)[5]) {
        if (GSd && GSd[li] > 0)    // Doppler cell (NEXT-1): weighted sums
            finalize_cell_dop(L.c[li], s5[0], s5[1], s5[2], s5[3], s5[4], L.Rp[li], mean, cov);
        else
            finalize_cell(L.c[li], s5[0], s5[1], s5[2], s5[3], s5[4], L.n[li], L.rho_p[li], w_pred, mean, cov);
    };
    auto single = [&](uint32_t li, uint32_t m = 1u) {      // few runs: one lane sums them in list order
        const uint32_t* pl = plist + L.ps[li];
        const double* ps = ppart[pl[0]].s;
        double s5[5] = {ps[0], ps[1], ps[2], ps[3], ps[4]};
        for (uint32_t q = 1; q < m; ++q) {
            const double* pq = ppart[pl[q]].s;
#pragma unroll
            for (int i = 0; i < 5; ++i) s5[i] += pq[i];
        }
        finalize(li, s5);
    };
    for_run_entries<kBatch, kMoGroup, kBatch ? kMoSmall : 1>(L.np, Lc, [&](uint32_t li, uint32_t m) {
        const uint32_t* pl = plist + L.ps[li];
        double s5[5] = {0, 0, 0, 0, 0};
        for (uint32_t q = gl; q < m; q += kMoGroup) {
            const double* ps = ppart[pl[q]].s;
#pragma unroll
            for (int i = 0; i < 5; ++i) s5[i] += ps[i];
        }
        if (m > 1) {
#pragma unroll
            for (int d = kMoGroup / 2; d; d >>= 1)
#pragma unroll
                for (int i = 0; i < 5; ++i) s5[i] += __shfl_xor_sync(gmask, s5[i], d, kMoGroup);
        }
        if (gl == 0) finalize(li, s5);
    }, single);
}

// Split of a cell's birth slots / born mass into the associated and unassociated sets (NEXT-1, A-36):
// nu_A = floor(p_A nb + 1/2), R_bA = floor(R_b p_A) (fp64), 0 if nu_A = 0, R_b if nu_A = nb.
__device__ __forceinline__ void birth_assoc_split(uint64_t Rb, uint32_t nb, float pA, uint32_t& nA, uint64_t& RbA)
{
    uint32_t na = (uint32_t)floor(__dadd_rn(__dmul_rn((double)pA, (double)nb), 0.5));
    if (na > nb) na = nb;
    uint64_t ra = __double2ull_rz(__dmul_rn(__ull2double_rn(Rb), (double)pA));
    if (na == 0) ra = 0;
    else if (na == nb) ra = Rb;
    nA = na;
    RbA = ra;
}

// New-born particles (Alg. 5): work items of <= 256 birth slots of one cell; each warp takes a
// contiguous range of items.  State from the slot's Philox draw; copies as for persistent members.
// dpA / ddop: the Doppler grid of the cycle (NEXT-1) or nullptr: slots r < nu_A of a cell with p_A > 0
// form the associated set (velocity from p(x | z)), sharing R_bA; the rest share R_b - R_bA (A-36).
__global__ __launch_bounds__(256) void k_births(CellList L, NextState out, BirthDebug bdbg,
                                                const DevScalars* __restrict__ sc, FilterConst fc, int64_t k,
                                                const float* __restrict__ dpA, const float4* __restrict__ ddop)
{
    PDL_ENTER();
    const int tid = threadIdx.x, lane = tid & 31;
    const RsConst rc = make_rsconst(sc, fc.nu);
    const int par = (int)(k & 1);
    out.s += fc.lo_cap - sc->o_base[par ^ 1];                     // global output -> local slot
    const uint64_t Ppre = sc->Ppre;                                // joint prefix of the shards below
    const uint32_t n_items = sc->n_items, Lc = sc->Lc;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    const uint32_t per = (n_items + nwarps - 1) / nwarps;
    uint32_t q = gw * per;
    const uint32_t q_end = min(q + per, n_items);
    if (q >= q_end) return;
    uint32_t li = warp_last_le(0u, Lc, q, [&](uint32_t i) { return L.it[i]; });
    uint32_t sub = q - L.it[li];
    while (true) {
        const uint32_t c = L.c[li], n = L.n[li], start = L.start[li], nb = L.nb[li];
        const uint64_t P = Ppre + L.P[li];
        const uint32_t r0 = sub * kItem, m = min(kItem, nb - r0);
        const uint64_t bb = L.bb[li];
        const uint32_t rbm = L.rb[li], sb = L.sb[li];
        const uint64_t PB = P + L.Rp[li];
        const uint32_t jbase = start + sb + n;
        uint32_t nA = 0;                                              // associated slots (NEXT-1)
        uint64_t RbA = 0, bbA = 0, bbB = bb;
        uint32_t rbA = 0, rbB = rbm;
        float4 dz = make_float4(0.f, 0.f, 0.f, 0.f);
        if (dpA) {
            const float pa = dpA[c];
            if (pa > 0.0f) {
                birth_assoc_split((uint64_t)nb * bb + rbm, nb, pa, nA, RbA);
                if (nA) { bbA = RbA / nA; rbA = (uint32_t)(RbA % nA); dz = ddop[c]; }
                const uint32_t nB = nb - nA;
                const uint64_t RbB = (uint64_t)nb * bb + rbm - RbA;
                if (nB) { bbB = RbB / nB; rbB = (uint32_t)(RbB % nB); }
            }
        }
        // fixed-point joint CDF of slot r within the cell's births
        auto slotQ = [&](uint32_t r) -> uint64_t {
            if (r < nA) return (uint64_t)r * bbA + min(r, rbA);
            const uint32_t rr = r - nA;
            return RbA + (uint64_t)rr * bbB + min(rr, rbB);
        };
        const uint32_t cg = c + fc.c_off;                             // global cell
        const uint32_t col = cg % (uint32_t)fc.W, row = cg / (uint32_t)fc.W;
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
            float bvx, bvy;
            if (r < nA) {                                             // associated: p(x | z), Eq. 74 (A-36)
                const float sr = __fmaf_rn(dz.w, n0, dz.z);
                const float st = __fmul_rn(fc.sigma_b, n1);
                bvx = __fmaf_rn(sr, dz.x, -__fmul_rn(st, dz.y));
                bvy = __fmaf_rn(sr, dz.y, __fmul_rn(st, dz.x));
            } else {
                bvx = __fmul_rn(fc.sigma_b, n0); bvy = __fmul_rn(fc.sigma_b, n1);
            }
            if (fc.v_max > 0.0f) {
                bvx = fminf(fmaxf(bvx, -fc.v_max), fc.v_max);
                bvy = fminf(fmaxf(bvy, -fc.v_max), fc.v_max);
            }
            if (valid && bdbg.x) { bdbg.x[s] = bx; bdbg.y[s] = by; bdbg.vx[s] = bvx; bdbg.vy[s] = bvy; }
            if (rc.W) {
                const uint64_t Q0 = PB + slotQ(r);
                const uint32_t F0 = valid ? fcount(Q0, rc) : 0u;
                uint32_t F1 = __shfl_down_sync(0xffffffffu, F0, 1);
                if (valid && (lane == 31 || t + lane + 1 == m)) F1 = fcount(PB + slotQ(r + 1), rc);
                write_copies(valid, F0, F1, bx, by, bvx, bvy, jbase + r, out);
            }
        }
        if (++q >= q_end) break;
        if (++sub < (nb + kItem - 1) / kItem) continue;
        sub = 0;
        li = warp_last_le(li + 1, Lc, q, [&](uint32_t i) { return L.it[i]; });
        sub = q - L.it[li];
    }
}

// New-born particles, one thread per birth SLOT (lists where most cells get one or two slots -- the
// exact filter spreads nu_b over the whole grid, so k_births' per-cell work items would leave most lanes
// idle).  Slot s belongs to the last list entry with sb <= s; same draws, state and joint CDF as
// k_births (no Doppler split); copies written by the slot's own thread.
__global__ __launch_bounds__(256) void k_births_slots(CellList L, NextState out, BirthDebug bdbg,
                                                      const DevScalars* __restrict__ sc, FilterConst fc, int64_t k)
{
    PDL_ENTER();
    const RsConst rc = make_rsconst(sc, fc.nu);
    const int par = (int)(k & 1);
    out.s += fc.lo_cap - sc->o_base[par ^ 1];
    const uint64_t Ppre = sc->Ppre;
    const uint32_t Lc = sc->Lc;
    const uint32_t ns = (uint32_t)sc->s_total;
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = Lc;                                   // last entry with sb <= s
        while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (L.sb[m] <= s) lo = m; else hi = m; }
        const uint32_t li = lo;
        const uint32_t c = L.c[li], nb = L.nb[li], sb = L.sb[li];
        if (s - sb >= nb) continue;                                 // (not reached: slots are dense)
        const uint32_t r = s - sb;
        const uint64_t bb = L.bb[li];
        const uint32_t rbm = L.rb[li];
        const uint64_t PB = Ppre + L.P[li] + L.Rp[li];
        const uint32_t cg = c + fc.c_off;
        const uint32_t col = cg % (uint32_t)fc.W, row = cg / (uint32_t)fc.W;
        const float colf = (float)col, rowf = (float)row;
        const float cx1 = __fadd_rn(colf, 1.0f), cy1 = __fadd_rn(rowf, 1.0f);
        const Philox4 d = draw(fc.seed, s, k, STAGE_BIRTH);
        float bx = __fadd_rn(colf, unit24(d.r0));
        float by = __fadd_rn(rowf, unit24(d.r1));
        if (bx >= cx1) bx = __int_as_float(__float_as_int(cx1) - 1);
        if (by >= cy1) by = __int_as_float(__float_as_int(cy1) - 1);
        float n0, n1;
        box_muller(d.r2, d.r3, n0, n1);
        float bvx = __fmul_rn(fc.sigma_b, n0), bvy = __fmul_rn(fc.sigma_b, n1);
        if (fc.v_max > 0.0f) {
            bvx = fminf(fmaxf(bvx, -fc.v_max), fc.v_max);
            bvy = fminf(fmaxf(bvy, -fc.v_max), fc.v_max);
        }
        if (bdbg.x) { bdbg.x[s] = bx; bdbg.y[s] = by; bdbg.vx[s] = bvx; bdbg.vy[s] = bvy; }
        if (rc.W) {
            const uint64_t Q0 = PB + (uint64_t)r * bb + min(r, rbm);
            const uint64_t Q1 = Q0 + bb + (r < rbm ? 1u : 0u);
            const uint32_t F0 = fcount(Q0, rc), F1 = fcount(Q1, rc);
            DOG_ASSERT(F0 <= F1 && F1 <= fc.nu);
            const uint32_t J = L.start[li] + sb + L.n[li] + r;
            for (uint32_t o = F0; o < F1; ++o) {
                out.s[o] = make_float4(bx, by, bvx, bvy);
                if (out.jidx) out.jidx[o] = J;
            }
        }
    }
}

}  // namespace dog
