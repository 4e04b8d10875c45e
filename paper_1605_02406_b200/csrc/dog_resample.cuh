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
    const double f = (double)w / (double)rp;                   // one fp64 division per cell
    const double mx = s0 * f, my = s1 * f;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(s2 * f - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(s3 * f - my * my);
    cov[3 * (size_t)c + 2] = (float)(s4 * f - mx * my);
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
    const double f = 1.0 / (double)Rp;
    const double mx = s0 * f, my = s1 * f;
    mean[c] = make_float2((float)mx, (float)my);
    cov[3 * (size_t)c] = (float)(s2 * f - mx * mx);
    cov[3 * (size_t)c + 1] = (float)(s3 * f - my * my);
    cov[3 * (size_t)c + 2] = (float)(s4 * f - mx * my);
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
static_assert(kRtItems % 8 == 0, "16-byte vector loads of the tile arrays");
constexpr uint32_t kRtShortSpan = 8;                                  // phase R: longer runs combined by a warp

#ifndef RT_RUNCACHE
#define RT_RUNCACHE 256
#endif
constexpr int kRtRunCache = RT_RUNCACHE;                                      // runs whose RunF sits in smem

// Per run, what the copy pass needs to place member r = pre + k (k = position - first): F(Q_r) =
// ceil(y(r)) with y(r) = y0 + r d1 for r <= rpm and yR + (r - rpm) d2 beyond (Q is linear in r on both
// pieces, steps bp + 1 and bp; yR = y0 + rpm d1, d2 = d1 - nu/W).
struct RunF {
    double y0, d1;
    uint32_t pre, rpm, first, pad;
};
static_assert(sizeof(RunF) == 32, "RunF: two per 64-byte line");

struct RtSmem {   // dynamic shared memory of k_resample_tiles (~9.7 KB)
    RunF rf[kRtRunCache];
    uint32_t starts[kSortTile / 32];   // bitmap of run starts over the tile's sorted positions
    uint32_t dir[kSortTile / 32];      // bitmap over the tile's runs: kRunDirect (no run sums needed)
    uint32_t dop[kSortTile / 32];      // bitmap over the tile's runs: likelihood-weighted cell (k_resample_dopp)
    uint16_t long_run[kSortTile / 16]; // runs of >= 16 members (summed warp-wide)
    uint32_t n_long;
    uint32_t sentinel_run;             // index of the run outside the grid, or 0xFFFFFFFF
};
constexpr size_t kRtSmemBytes = sizeof(RtSmem);

// Q of member mr of a run's cell: P + mr bp + min(mr, rpm) (even split of the cell's R_p, A-23).
__device__ __forceinline__ uint64_t member_Q(const RunQ& q, uint32_t mr)
{
    return q.P + (uint64_t)mr * q.bp + min(mr, q.rpm);
}

// ceil(y) clamped to [0, nu] when y is further than `margin` from an integer; otherwise *amb is set (the
// caller settles it with exact products).  The per-run linear estimates are within ~nu 2^-50 of the exact
// value, so margin = max(2^-22, nu 2^-48) keeps every accepted ceiling exact.
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

// Warp-cooperative write of the copies of 32 members (lanes) whose output ranges [F0_l, F0_l + c_l) are
// arbitrary (members of different runs own ranges far apart): the copies are numbered compactly over
// the lanes (exclusive prefix of c), and 32 consecutive copy numbers are written per round; the owner of
// copy o is the last lane whose prefix is <= o (a 5-step shuffle search).  Consecutive copies of a run
// are consecutive outputs, so the stores coalesce within runs; the rounds are balanced whatever the copy
// counts (a member can own hundreds of outputs).
template <bool kDbg>
__device__ __forceinline__ void write_compact(uint32_t c, uint32_t F0, const float4& X, uint32_t J, NextState& out,
                                              uint32_t nu)
{
    const int lane = threadIdx.x & 31;
    if (__reduce_max_sync(0xffffffffu, c) <= 2u) {         // the common case: each lane writes its own
        if (c > 0u) {                                      // (consecutive members of a run own
            DOG_ASSERT(F0 < nu);                           //  consecutive outputs: coalesced)
            out.s[F0] = X;
            if (kDbg) out.jidx[F0] = J;
        }
        if (c > 1u) {
            DOG_ASSERT(F0 + 1u < nu);
            out.s[F0 + 1u] = X;
            if (kDbg) out.jidx[F0 + 1u] = J;
        }
        return;
    }
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t ex = incl - c;
    for (uint32_t o0 = 0; o0 < total; o0 += 32) {
        const uint32_t o = o0 + lane;
        int own = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, ex, own + step);
            if (e <= o) own += step;
        }
        const uint32_t dst = __shfl_sync(0xffffffffu, F0, own) + (o - __shfl_sync(0xffffffffu, ex, own));
        const float4 V = make_float4(__shfl_sync(0xffffffffu, X.x, own), __shfl_sync(0xffffffffu, X.y, own),
                                     __shfl_sync(0xffffffffu, X.z, own), __shfl_sync(0xffffffffu, X.w, own));
        const uint32_t jj = kDbg ? __shfl_sync(0xffffffffu, J, own) : 0u;
        if (o < total) {
            DOG_ASSERT(dst < nu);
            out.s[dst] = V;
            if (kDbg) out.jidx[dst] = jj;
        }
    }
    (void)nu;
}

// Persistent particles, one block per sort tile: the tile's predicted state arrives in sorted (cell)
// order (k_predict_sort), so warp w walks sorted positions [512 w, 512 w + 512) 32 at a time, lanes on
// consecutive positions -- every read is coalesced.  Member r of its cell owns the outputs
// [F(Q_r), F(Q_{r+1})) (A-24): F from the run's linear estimate, exact whenever the estimate is clear of an
// integer, else from exact 128-bit products (dog_fcount.cuh); the warp writes its 32 members' copies
// with write_compact.  The run of a position comes from a bitmap of run starts (popcount), the run's F
// parameters from shared memory.  (The velocity moments are summed per cell by k_moments.)
template <bool kDbg>
__global__ __launch_bounds__(kRtThreads) void k_resample_tiles(
    const uint16_t* __restrict__ lperm, TilePairs tp, const float2* __restrict__ pxy, const float2* __restrict__ pv,
    CellList L, NextState out, uint32_t* __restrict__ perm_dbg, MomPartial* __restrict__ ppart,
    const DevScalars* sc, FilterConst fc, int par, const uint64_t* __restrict__ dopGS, uint32_t mo_direct)
{
    PDL_ENTER();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    RtSmem& S = *reinterpret_cast<RtSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = blockIdx.x, base = t * kSortTile;     // this tile's slot in the per-tile arrays
    const RsConst rc = make_rsconst(sc, fc.nu, fc.force_exact != 0);
    const uint32_t n_lo = scrd(sc->n_lo), n_loc = n_lo + scrd(sc->n_own[par]) + scrd(sc->n_hi);
    const uint32_t pbase = fc.lo_cap - n_lo + base;                // its first particle
    // next-cycle own particles start at lo_cap: global output o -> slot lo_cap + o - F(P'_shard)
    out.s += fc.lo_cap - scrd(sc->o_base[par ^ 1]);
    if (rc.W == 0 && fc.world == 1) {   // empty world (A-26): every next particle goes to the sentinel
        for (uint32_t i = blockIdx.x * blockDim.x + tid; i < fc.nu; i += gridDim.x * blockDim.x) {
            out.s[i] = make_float4(kSentinelPos, kSentinelPos, 0.0f, 0.0f);
            if (kDbg) out.jidx[i] = 0xFFFFFFFFu;
        }
    }
    const uint32_t n = n_loc > base ? min((uint32_t)kSortTile, n_loc - base) : 0u;
    if (n == 0) return;
    const uint32_t nd = tp.nd[t];
    const RunInfo* __restrict__ runs = tp.run + base;
    const uint64_t Ppre = scrd(sc->Ppre);                          // joint prefix of the shards below
    // ---- run starts (bitmap) and the runs' F parameters
    for (uint32_t w = tid; w < kSortTile / 32; w += kRtThreads) { S.starts[w] = 0u; S.dir[w] = 0u; S.dop[w] = 0u; }
    if (tid == 0) S.sentinel_run = tp.key[base + nd - 1] >= fc.C ? nd - 1 : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t r = tid; r < nd; r += kRtThreads) {
        const uint32_t f = tp.first[base + r];
        atomicOr(&S.starts[f >> 5], 1u << (f & 31u));
        if (r < (uint32_t)kRtRunCache && r != S.sentinel_run) {   // (the run outside the grid has no RunInfo)
            const RunQ q = run_q(runs[r], L, Ppre);
            if (q.direct) atomicOr(&S.dir[r >> 5], 1u << (r & 31u));
            if (dopGS && dopGS[q.li] > 0) atomicOr(&S.dop[r >> 5], 1u << (r & 31u));
            RunF x;
            x.y0 = __fma_rn((double)q.P, rc.nu_over_W, -rc.U_frac);
            x.d1 = __dmul_rn((double)(q.bp + 1u), rc.nu_over_W);
            x.pre = q.pre; x.rpm = q.rpm; x.first = f; x.pad = 0u;
            if (r < (uint32_t)kRtRunCache) S.rf[r] = x;
        }
    }
    __syncthreads();
    const uint32_t srun = S.sentinel_run;
    const double margin = fc.force_exact ? 1.0 : fast_ceil_margin(fc.nu);   // 1.0: every estimate ambiguous
    // ---- copies: warp w, sorted positions [512 w, 512 w + 512), 32 per round
    constexpr uint32_t kSpan = kSortTile / (kRtThreads / 32);
    const uint32_t w0 = warp * kSpan;                      // (warps beyond n skip the loop, not the barrier)
    int jprev = -1;                                         // run of position w0 - 1
    {
        uint32_t c = 0;
        for (uint32_t k = lane; k < w0 / 32; k += 32) c += __popc(S.starts[k]);
        jprev += (int)__reduce_add_sync(0xffffffffu, c);
    }
    const uint32_t wend = w0 < n ? min(w0 + kSpan, n) : w0;
    for (uint32_t p0 = w0; p0 < wend; p0 += 32) {
        const uint32_t p = p0 + lane;
        const uint32_t word = S.starts[p0 >> 5];
        const uint32_t j = (uint32_t)(jprev + (int)__popc(lane == 31 ? word : (word & ((2u << lane) - 1u))));
        jprev += (int)__popc(word);
        const bool mem = p < wend && j != srun;
        float2 XY = make_float2(0.f, 0.f), V = XY;
        if (mem) { XY = pxy[pbase + p]; V = pv[pbase + p]; }   // coalesced, issued early
        // member mr owns [F(Q_mr), F(Q_mr+1)): each lane settles F(Q_mr) (linear estimate, exact fallback);
        // F(Q_mr+1) is the next lane's value when it holds the run's next member
        uint32_t F0 = 0, Jd = 0, mr = 0;
        RunF x{};
        RunQ qf{};
        const bool cached = j < (uint32_t)kRtRunCache;       // else (run-heavy tiles): F from the cell parameters
        bool memb = mem;                                    // members of likelihood-weighted cells: k_resample_dopp
        if (mem) {
            if (cached && dopGS && ((S.dop[j >> 5] >> (j & 31u)) & 1u)) {
                memb = false;
            } else if (cached) {
                x = S.rf[j];
                mr = x.pre + (p - x.first);
                const double y0 = mr <= x.rpm ? __fma_rn((double)mr, x.d1, x.y0)
                                              : __fma_rn((double)(mr - x.rpm), x.d1 - rc.nu_over_W, __fma_rn((double)x.rpm, x.d1, x.y0));
                bool amb = false;
                F0 = fast_ceil(y0, rc.nu, margin, amb);
                if (amb) F0 = fcount(member_Q(run_q(runs[j], L, Ppre), mr), rc);   // rare: exact products
            } else {
                qf = run_q(runs[j], L, Ppre);
                if (qf.direct) atomicOr(&S.dir[j >> 5], 1u << (j & 31u));
                if (dopGS && dopGS[qf.li] > 0) {
                    memb = false;
                    atomicOr(&S.dop[j >> 5], 1u << (j & 31u));
                } else {
                    mr = qf.pre + (p - tp.first[base + j]);
                    F0 = fcount(member_Q(qf, mr), rc);
                }
            }
            if (kDbg && memb) {
                const RunQ q = run_q(runs[j], L, Ppre);
                Jd = L.start[q.li] + L.sb[q.li] + mr;
                perm_dbg[L.start[q.li] + mr] = pbase + lperm[base + p];
            }
        }
        const uint32_t Fn = __shfl_down_sync(0xffffffffu, F0, 1);
        const uint32_t jn = __shfl_down_sync(0xffffffffu, memb ? j : 0xFFFFFFFFu, 1);
        uint32_t c = 0;
        if (memb) {
            uint32_t F1 = Fn;
            if (lane == 31 || jn != j) {                    // the run's last member in this round
                if (cached) {
                    const double y1 = mr < x.rpm ? __fma_rn((double)(mr + 1u), x.d1, x.y0)
                                                 : __fma_rn((double)(mr + 1u - x.rpm), x.d1 - rc.nu_over_W,
                                                            __fma_rn((double)x.rpm, x.d1, x.y0));
                    bool amb = false;
                    F1 = fast_ceil(y1, rc.nu, margin, amb);
                    if (amb) {
                        const RunQ q = run_q(runs[j], L, Ppre);
                        F1 = fcount(member_Q(q, mr) + q.bp + (mr < q.rpm ? 1u : 0u), rc);
                    }
                } else {
                    F1 = fcount(member_Q(qf, mr) + qf.bp + (mr < qf.rpm ? 1u : 0u), rc);
                }
            }
            DOG_ASSERT(F0 <= F1 && F1 <= fc.nu);
            c = F1 - F0;
        }
        write_compact<kDbg>(c, F0, make_float4(XY.x, XY.y, V.x, V.y), Jd, out, fc.nu);
    }
    // ---- velocity sums per run (Eqs. 81-84; k_moments combines a cell's runs in tile order), from the
    //      sorted predicted velocities just read (L1 / L2): runs of >= 16 members by a warp each (lanes
    //      strided, fixed butterfly), shorter runs by one thread each in member order -- deterministic.
    auto run_bounds = [&](uint32_t r, uint32_t& f, uint32_t& e) {
        f = tp.first[base + r];
        e = r + 1 < nd ? (uint32_t)tp.first[base + r + 1] : n;
    };
    auto warp_run = [&](uint32_t r, uint32_t f, uint32_t e) {
        double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (uint32_t q = f + lane; q < e; q += 32) {
            const float2 V = pv[pbase + q];
            const double a = (double)V.x, b = (double)V.y;
            s5[0] += a; s5[1] += b; s5[2] += a * a; s5[3] += b * b; s5[4] += a * b;
        }
#pragma unroll
        for (int dd = 16; dd; dd >>= 1)
#pragma unroll
            for (int i = 0; i < 5; ++i) s5[i] += __shfl_xor_sync(0xffffffffu, s5[i], dd);
        if (lane == 0) {
            MomPartial mp;
#pragma unroll
            for (int i = 0; i < 5; ++i) mp.s[i] = s5[i];
            ppart[base + r] = mp;
        }
    };
    auto thread_run = [&](uint32_t r, uint32_t f, uint32_t e) {
        double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (uint32_t q = f; q < e; ++q) {
            const float2 V = pv[pbase + q];
            const double a = (double)V.x, b = (double)V.y;
            s5[0] += a; s5[1] += b; s5[2] += a * a; s5[3] += b * b; s5[4] += a * b;
        }
        MomPartial mp;
#pragma unroll
        for (int i = 0; i < 5; ++i) mp.s[i] = s5[i];
        ppart[base + r] = mp;
    };
    constexpr uint32_t nw = kRtThreads / 32;
    auto dop_run = [&](uint32_t r) -> bool {                // weighted runs: k_resample_dopp sums them
        if (!dopGS) return false;
        if (r < (uint32_t)kRtRunCache) return ((S.dop[r >> 5] >> (r & 31u)) & 1u) != 0u;
        return dopGS[runs[r].li & ~kRunDirect] > 0;
    };
    if (!mo_direct) {   // few, long runs: warps walk the runs directly (no barrier)
        for (uint32_t r = warp; r < nd; r += nw) {
            uint32_t f, e;
            run_bounds(r, f, e);
            if (r != srun && e - f >= 16u && !dop_run(r)) warp_run(r, f, e);
        }
        for (uint32_t r = tid; r < nd; r += kRtThreads) {
            uint32_t f, e;
            run_bounds(r, f, e);
            if (r != srun && e - f < 16u && !dop_run(r)) thread_run(r, f, e);
        }
        return;
    }
    // long-list cycles (thousands of short runs per tile): thread per run; the runs of cells k_moments sums
    // directly (kRunDirect) are skipped, the (at most 256) long ones listed, then summed warp-wide
    if (tid == 0) S.n_long = 0u;
    __syncthreads();                                        // S.dir complete (every run has a member here)
    for (uint32_t r = tid; r < nd; r += kRtThreads) {
        if (r == srun || ((S.dir[r >> 5] >> (r & 31u)) & 1u) || ((S.dop[r >> 5] >> (r & 31u)) & 1u)) continue;
        uint32_t f, e;
        run_bounds(r, f, e);
        if (e - f >= 16u) S.long_run[atomicAdd(&S.n_long, 1u)] = (uint16_t)r;
        else thread_run(r, f, e);
    }
    __syncthreads();
    for (uint32_t w = (uint32_t)warp; w < S.n_long; w += nw) {
        const uint32_t r = S.long_run[w];
        uint32_t f, e;
        run_bounds(r, f, e);
        warp_run(r, f, e);
    }
}

// Velocity moments per cell (Eqs. 81-84): the cell's run sums combined in tile order (k_pair_sort left
// the run list in that order) in a fixed summation order.  Groups of 8 lanes take one cell each.
constexpr int kMoGroup = 8;
constexpr int kMoSmall = 4;   // kBatch (exact filter): cells with <= 4 runs summed by one lane each

// Velocity sums of the members of run v (tile << 12 | run) from the sorted predicted velocities (member
// order); used for cells of at most kMoDirect particles, whose runs' sums k_resample_tiles skips.
__device__ __forceinline__ void run_vsums(const float2* __restrict__ v0, TilePairs tp, uint32_t v, double (&s5)[5])
{
    const uint32_t cnt = (uint32_t)tp.cnt[v] + 1u;
    const float2* __restrict__ r = v0 + (v & ~0xFFFu) + tp.first[v];
    for (uint32_t k = 0; k < cnt; ++k) {
        const float2 V = r[k];
        const double a = (double)V.x, b = (double)V.y;
        s5[0] += a; s5[1] += b; s5[2] += a * a; s5[3] += b * b; s5[4] += a * b;
    }
}

template <bool kBatch>
__global__ __launch_bounds__(256) void k_moments(CellList L, TilePairs tp, const uint32_t* __restrict__ plist,
                                                 const float2* __restrict__ pv, const MomPartial* __restrict__ ppart,
                                                 float2* __restrict__ mean, float* __restrict__ cov, const DevScalars* sc,
                                                 FilterConst fc, const uint64_t* __restrict__ GSd)
{
    PDL_ENTER();
    const int lane = threadIdx.x & 31, gl = lane & (kMoGroup - 1);
    const uint32_t gmask = 0xFFu << (lane & ~(kMoGroup - 1));
    const uint32_t Lc = scrd(sc->Lc);
    const float w_pred = scrd(sc->w_pred);
    const float2* __restrict__ v0 = pv + (fc.lo_cap - scrd(sc->n_lo));   // sorted position p of tile t: v0[t 4096 + p]
    auto dop = [&](uint32_t li) { return GSd && GSd[li] > 0; };
    auto direct = [&](uint32_t li) { return kBatch && !dop(li) && L.n[li] <= kMoDirect; };
    auto finalize = [&](uint32_t li, const double (&s5)[5]) {
        if (dop(li))               // Doppler cell (NEXT-1): weighted sums
            finalize_cell_dop(L.c[li], s5[0], s5[1], s5[2], s5[3], s5[4], L.Rp[li], mean, cov);
        else
            finalize_cell(L.c[li], s5[0], s5[1], s5[2], s5[3], s5[4], L.n[li], L.rho_p[li], w_pred, mean, cov);
    };
    auto single = [&](uint32_t li, uint32_t m = 1u) {      // few runs: one lane sums them in list order
        const uint32_t* pl = plist + L.ps[li];
        double s5[5] = {0, 0, 0, 0, 0};
        const bool dir = direct(li);
        for (uint32_t q = 0; q < m; ++q) {
            if (dir) {
                run_vsums(v0, tp, pl[q], s5);
            } else {
                const double* pq = ppart[pl[q]].s;
#pragma unroll
                for (int i = 0; i < 5; ++i) s5[i] += pq[i];
            }
        }
        finalize(li, s5);
    };
    for_run_entries<kBatch, kMoGroup, kBatch ? kMoSmall : 1>(L.np, Lc, [&](uint32_t li, uint32_t m) {
        const uint32_t* pl = plist + L.ps[li];
        double s5[5] = {0, 0, 0, 0, 0};
        const bool dir = direct(li);
        for (uint32_t q = gl; q < m; q += kMoGroup) {
            if (dir) {
                run_vsums(v0, tp, pl[q], s5);
            } else {
                const double* ps = ppart[pl[q]].s;
#pragma unroll
                for (int i = 0; i < 5; ++i) s5[i] += ps[i];
            }
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
                                                const DevScalars* sc, FilterConst fc, int64_t k,
                                                const float* __restrict__ dpA, const float4* __restrict__ ddop)
{
    PDL_ENTER();
    const int tid = threadIdx.x, lane = tid & 31;
    const RsConst rc = make_rsconst(sc, fc.nu, fc.force_exact != 0);
    const int par = (int)(k & 1);
    out.s += fc.lo_cap - scrd(sc->o_base[par ^ 1]);                     // global output -> local slot
    const uint64_t Ppre = scrd(sc->Ppre);                                // joint prefix of the shards below
    const uint32_t n_items = scrd(sc->n_items), Lc = scrd(sc->Lc);
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    const uint32_t per = (n_items + nwarps - 1) / nwarps;
    uint32_t q = gw * per;
    const uint32_t q_end = min(q + per, n_items);
    if (q >= q_end) return;
    uint32_t li = warp_last_le(0u, Lc, q, [&](uint32_t i) { return L.it[i]; });
    uint32_t sub = q - L.it[li];
    while (true) {
        const BirthRec R = L.brec[li];                                // an entry with items has n_b > 0
        const uint32_t c = R.c, nb = R.nb;
        const uint32_t r0 = sub * kItem, m = min(kItem, nb - r0);
        const uint64_t bb = R.bb;
        const uint32_t rbm = R.rb, sb = R.sb;
        const uint64_t PB = Ppre + R.PB;
        const uint32_t jbase = out.jidx ? L.start[li] + sb + L.n[li] : 0u;   // joint index (debug dump)
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
// The exact filter with a likelihood (A-38): in a cell where a measurement occurred and p_A > 0, the
// first nu_A = floor(pi nb + 1/2) slots draw the radial velocity from the posterior given z; the weights
// stay the single even split of R_b (the associated set's part of it is R_bA).  pA == nullptr: off.
struct BirthLik {
    const float* pA;
    const float4* obs;
    const float4* lik;
    const float* pic;
};

__global__ __launch_bounds__(256) void k_births_slots(CellList L, NextState out, BirthDebug bdbg,
                                                      const DevScalars* sc, FilterConst fc, int64_t k, BirthLik bl)
{
    PDL_ENTER();
    const RsConst rc = make_rsconst(sc, fc.nu, fc.force_exact != 0);
    const int par = (int)(k & 1);
    out.s += fc.lo_cap - scrd(sc->o_base[par ^ 1]);
    const uint64_t Ppre = scrd(sc->Ppre);
    const uint32_t Lc = scrd(sc->Lc);
    const uint32_t ns = (uint32_t)scrd(sc->s_total);
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t s0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); s0 < ns; s0 += gridDim.x * blockDim.x) {
        // last entry with sb <= s: the warp brackets its 32 slots with two 32-ary searches, then each lane
        // bisects the (short) bracket
        // (band contexts: slots are global, so those below the band's first entry belong to other bands)
        const uint32_t s = s0 + lane;
        if (Lc == 0u) continue;
        const uint32_t sb0 = L.sb[0], s_last = min(s0 + 31u, ns - 1u);
        if (s_last < sb0) continue;                                 // warp-uniform
        const uint32_t l0 = warp_last_le(0u, Lc, max(s0, sb0), [&](uint32_t i) { return L.sb[i]; });
        const uint32_t l1 = warp_last_le(l0, Lc, s_last, [&](uint32_t i) { return L.sb[i]; });
        if (s >= ns || s < sb0) continue;
        uint32_t lo = l0, hi = l1 + 1u;
        while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (L.sb[m] <= s) lo = m; else hi = m; }
        const uint32_t li = lo;
        if (s - L.sb[li] >= L.nb[li]) continue;                     // slots of another band's cells
        const BirthRec R = L.brec[li];
        const uint32_t c = R.c, nb = R.nb, sb = R.sb;
        const uint32_t r = s - sb;
        const uint64_t bb = R.bb;
        const uint32_t rbm = R.rb;
        const uint64_t PB = Ppre + R.PB;
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
        if (bl.pA && bl.obs[c].x > 0.0f && bl.pA[c] > 0.0f) {
            uint32_t nA = (uint32_t)floor(__dadd_rn(__dmul_rn((double)bl.pic[c], (double)nb), 0.5));
            if (r < min(nA, nb)) {                                  // posterior radial velocity given z (A-38)
                const float4 z = bl.lik[c];
                const float sb2 = __fmul_rn(fc.sigma_b, fc.sigma_b), sd2 = __fmul_rn(z.w, z.w);
                const float mu_r = __fdiv_rn(__fmul_rn(z.z, sb2), __fadd_rn(sb2, sd2));
                const float s_r = __fdiv_rn(__fmul_rn(fc.sigma_b, z.w), __fsqrt_rn(__fadd_rn(sb2, sd2)));
                const float sr = __fmaf_rn(s_r, n0, mu_r);
                const float st = __fmul_rn(fc.sigma_b, n1);
                bvx = __fmaf_rn(sr, z.x, -__fmul_rn(st, z.y));
                bvy = __fmaf_rn(sr, z.y, __fmul_rn(st, z.x));
            }
        }
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
