// dog_doppler.cuh -- the Doppler / association branch of the cycle (Eqs. 69-80,
// P:1157-1232; A-34..A-36).  Measurement cells may carry a radial-velocity measurement
// (u, v_r, sd) with association probability p_A > 0.  Then:
//   * persistent members get w~ = g w_pred (Eq. 69) and w = p_A mu_A w~ + (1 - p_A) mu_Abar w_pred
//     (Eqs. 71-73): member j of the cell owns [Q_j, Q_{j+1}) of the cell's fixed-point mass R_p with
//     Q_j = floor(R_p G_j), G_j = fma(p_A, GS_j / GS, (1 - p_A) j / n) (A-35), GS_j the exclusive
//     prefix of the fixed-point likelihoods gfx = floor((g / g_max) 2^31) (A-34) in cell order, g_max
//     the cell's largest likelihood;
//   * the cell's nu_b birth slots split into nu_A associated slots (velocity from p(x | z)) and
//     nu_b - nu_A unassociated ones, sharing R_bA and R_b - R_bA (A-36).
// Weights are no longer uniform within a cell, so the closed-form per-run resampling of
// k_resample_tiles does not apply to its runs; this path uses
//   k_dopp_g       per tile: g of every member, the cell maxima g_max (integer atomicMax: order-free)
//   k_dopp_runs    per tile: gfx of every member, summed per run (integer atomics: order-free)
//   k_pair_sort    (its Doppler branch) per active cell: the runs' gfx sums in tile order -> exclusive
//                  prefixes, cell total GS, tile flags
//   k_resample_dopp per tile holding a Doppler cell's members, for the runs of such cells only: block
//                  prefix of gfx -> GS_j of every member -> Q_j, Q_{j+1} -> F(.) -> copies; weighted
//                  velocity sums per run for the moments.  k_resample_tiles takes every tile and skips
//                  those runs (closed form, even split for the others).
//   k_moments (its Doppler branch), k_births (the associated slots).
// Every floating-point step uses explicit round-to-nearest intrinsics in the oracle's operation order,
// so the next state is bit-identical to orc_step_doppler.
#pragma once
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_fcount.cuh"
#include "dog_resample.cuh"
#include "dog_sort.cuh"

namespace dog {

struct DopIn {
    const float4* dop;    // [C] (u_x, u_y, v_r, sd)
    const float* pA;      // [C] association probability (0: no Doppler in the cell)
    const float4* gate;   // [C] obs of the exact filter (A-38): only cells where a measurement occurred; or nullptr
};

// the association probability a member of cell `key` is weighted with (0: no likelihood)
__device__ __forceinline__ float din_pa(const DopIn& din, uint32_t key, uint32_t C)
{
    if (key >= C) return 0.0f;
    const float pa = din.pA[key];
    return (pa > 0.0f && din.gate && !(din.gate[key].x > 0.0f)) ? 0.0f : pa;
}

// Doppler likelihood g(z | x) of a predicted velocity (Eq. 69; A-34), f32
__device__ __forceinline__ float doppler_g(float vx, float vy, float4 d)
{
    const float e = __fsub_rn(__fmaf_rn(vx, d.x, __fmul_rn(vy, d.y)), d.z);
    const float t = __fdiv_rn(e, d.w);
    const float q = __fmul_rn(__fmul_rn(t, t), -0.5f);
    const float g = __fdiv_rn(exp_spec(q), __fmul_rn(d.w, 2.50662827463100050f));
    return g < 0x1.fffffep+127f ? g : 0x1.fffffep+127f;      // inf (and NaN) -> FLT_MAX: finite inputs only, see dog.h
}

// fixed point relative to the cell's largest likelihood: floor((g / g_max) 2^31) (A-34)
__device__ __forceinline__ uint32_t doppler_gfx(float g, float gmax)
{
    if (!(g > 0.0f) || !(gmax > 0.0f)) return 0u;
    return __float2uint_rz(__fmul_rn(__fdiv_rn(g, gmax), 2147483648.0f));
}

// Q_j = floor(R_p G_j) (A-35)
__device__ __forceinline__ uint64_t doppler_Q(uint64_t Rp, float pA, uint64_t GSj, uint64_t GS, uint32_t j, uint32_t n)
{
    const double pa = (double)pA;
    const double a = __ddiv_rn(__ull2double_rn(GSj), __ull2double_rn(GS));
    const double b = __dmul_rn(__dsub_rn(1.0, pa), __ddiv_rn((double)j, (double)n));
    const double G = __fma_rn(pa, a, b);
    return __double2ull_rz(__dmul_rn(__ull2double_rn(Rp), G));
}

// particles of tile t (input order) and its slot base in the local array, as in k_resample_tiles
__device__ __forceinline__ uint32_t tile_count(const DevScalars* sc, int par, uint32_t base)
{
    const uint32_t n_loc = scrd(sc->n_lo) + scrd(sc->n_own[par]) + scrd(sc->n_hi);
    return n_loc > base ? min((uint32_t)kSortTile, n_loc - base) : 0u;
}

// run of sorted position p among first[0..nd) (first[0] = 0)
__device__ __forceinline__ uint32_t run_of(const uint16_t* first, uint32_t nd, uint32_t p)
{
    uint32_t lo = 0, hi = nd;
    while (hi - lo > 1) { const uint32_t m = (lo + hi) >> 1; if (first[m] <= p) lo = m; else hi = m; }
    return lo;
}

// Warp walk over a tile's sorted positions (as k_resample_tiles): warp w takes [512 w, 512 w + 512), 32
// consecutive positions per round, lane-contiguous (coalesced); the run of a position from a bitmap of
// run starts (popcount).  Per round, values of the same run are combined by a segmented reduction
// (shuffle doubling; runs are contiguous), whose result sits in the run's first lane of the round.
struct DopWalkSmem {
    uint32_t starts[kSortTile / 32];   // run starts over the tile's sorted positions
    uint32_t lik[kSortTile / 32];      // runs of a cell with a likelihood (din_pa > 0)
    uint32_t key[kSortTile];           // cell of each run (C: outside)
};

// loads the run starts and keys; returns false (block-uniform) if no run of the tile has a likelihood
__device__ __forceinline__ bool dop_walk_setup(DopWalkSmem& S, TilePairs tp, uint32_t base, uint32_t nd,
                                               const DopIn& din, uint32_t C)
{
    for (uint32_t w = threadIdx.x; w < kSortTile / 32; w += blockDim.x) { S.starts[w] = 0u; S.lik[w] = 0u; }
    __syncthreads();
    bool any = false;
    for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x) {
        const uint32_t f = tp.first[base + r], key = tp.key[base + r];
        atomicOr(&S.starts[f >> 5], 1u << (f & 31u));
        S.key[r] = key;
        if (din.pA && din_pa(din, key, C) > 0.0f) {
            atomicOr(&S.lik[r >> 5], 1u << (r & 31u));
            any = true;
        }
    }
    return __syncthreads_or(any);
}

template <typename T, typename Op>
__device__ __forceinline__ T seg_reduce(T v, uint32_t j, Op op)   // lane l: op over [l, end of its run)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const T o = __shfl_down_sync(0xffffffffu, v, dd);
        const uint32_t oj = __shfl_down_sync(0xffffffffu, j, dd);
        if (lane + dd < 32 && oj == j) v = op(v, o);
    }
    return v;
}

// calls body(p, j, lane_valid) for the positions of this warp, 32 per round (warp-uniform calls)
template <typename F>
__device__ __forceinline__ void dop_walk(const DopWalkSmem& S, uint32_t n, F&& body)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr uint32_t kSpan = kSortTile / 8;
    const uint32_t w0 = (uint32_t)warp * kSpan;
    int jprev = -1;
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
        body(p, j, p < wend);
    }
}

// ---- k_dopp_g: the likelihood g of every member of a cell with a likelihood (f32 bits per sorted position,
//      in gfx_out; 0 elsewhere in such tiles) and the cell's largest g (gmax[cell], integer atomicMax on
//      the bits of a nonnegative float: order-free; one per run and round).  gmax must be zero on entry.
__global__ __launch_bounds__(256) void k_dopp_g(TilePairs tp, const float2* __restrict__ pv, DopIn din,
                                                uint32_t* __restrict__ gmax, uint32_t* __restrict__ gfx_out,
                                                const DevScalars* sc, FilterConst fc, int par)
{
    PDL_ENTER();
    __shared__ DopWalkSmem S;
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    const uint32_t n = tile_count(sc, par, base);
    if (n == 0) return;
    const uint32_t nd = tp.nd[t];
    const uint32_t pbase = fc.lo_cap - scrd(sc->n_lo) + base;
    if (!dop_walk_setup(S, tp, base, nd, din, fc.C)) return;   // (tiles without one: nothing of them is read)
    const int lane = threadIdx.x & 31;
    dop_walk(S, n, [&](uint32_t p, uint32_t j, bool valid) {
        uint32_t gb = 0u, key = fc.C;
        if (valid) {
            key = S.key[j];
            if ((S.lik[j >> 5] >> (j & 31u)) & 1u) {         // a run of a cell with a likelihood
                const float2 V = pv[pbase + p];              // the tile's predicted state is in sorted order
                const float g = doppler_g(V.x, V.y, din.dop[key]);
                gb = g > 0.0f ? __float_as_uint(g) : 0u;        // NaN / 0 -> no weight
            }
            gfx_out[base + p] = gb;
        }
        const uint32_t mx = seg_reduce(gb, j, [](uint32_t a, uint32_t b) { return max(a, b); });
        const uint32_t jl = __shfl_up_sync(0xffffffffu, j, 1);
        if (valid && (lane == 0 || jl != j) && mx) atomicMax(&gmax[key], mx);
    });
}

// ---- k_dopp_runs: gfx = floor((g / g_max) 2^31) of every member of a cell with a likelihood, summed per run
//      (rg[run slot]; and per cell into gsc when given) by integer atomics (order-free, one per run and
//      round).  gfx_io holds g (k_dopp_g) on entry and gfx on exit.
__global__ __launch_bounds__(256) void k_dopp_runs(TilePairs tp, DopIn din, const uint32_t* __restrict__ gmax,
                                                   uint64_t* __restrict__ rg, uint8_t* __restrict__ tflag,
                                                   uint32_t* __restrict__ gfx_io, const DevScalars* sc,
                                                   FilterConst fc, int par, uint64_t* __restrict__ gsc)
{
    PDL_ENTER();
    __shared__ DopWalkSmem S;
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    if (threadIdx.x == 0) tflag[t] = 0;                      // set by k_pair_sort for Doppler tiles
    const uint32_t n = tile_count(sc, par, base);
    if (n == 0) return;
    const uint32_t nd = tp.nd[t];
    for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x) rg[base + r] = 0ull;
    if (!dop_walk_setup(S, tp, base, nd, din, fc.C)) return;   // no likelihood cell: gfx / rg of this tile unused
    const int lane = threadIdx.x & 31;
    dop_walk(S, n, [&](uint32_t p, uint32_t j, bool valid) {
        uint32_t gf = 0u, key = fc.C;
        if (valid) {
            key = S.key[j];
            if ((S.lik[j >> 5] >> (j & 31u)) & 1u)
                gf = doppler_gfx(__uint_as_float(gfx_io[base + p]), __uint_as_float(gmax[key]));
            gfx_io[base + p] = gf;                           // per sorted position, for k_resample_dopp
        }
        const uint64_t acc = seg_reduce((uint64_t)gf, j, [](uint64_t a, uint64_t b) { return a + b; });
        const uint32_t jl = __shfl_up_sync(0xffffffffu, j, 1);
        if (valid && (lane == 0 || jl != j) && acc) {
            atomicAdd((unsigned long long*)&rg[base + j], (unsigned long long)acc);
            if (gsc) atomicAdd((unsigned long long*)&gsc[key], (unsigned long long)acc);
        }
    });
}

// ---- k_resample_dopp: persistent members with per-member weights ---------------------------------------
constexpr int kRdItems = kSortTile / 256;   // 16 sorted positions per thread

struct RdSmem {
    MomPartial pa[256], pb[256];   // first / last run segment of each thread (spanning runs)
    uint64_t scan[9];
    uint16_t first[kSortTile + 1];
    uint32_t wrun[kSortTile / 32]; // bitmap over the tile's runs: a likelihood-weighted cell (GS > 0)
};
constexpr size_t kRdSmemBytes = sizeof(RdSmem);

__global__ __launch_bounds__(256, 4) void k_resample_dopp(TilePairs tp, const float2* __restrict__ pxy,
                                                       const float2* __restrict__ pv, CellList L, NextState out,
                                                       MomPartial* __restrict__ ppart, DopIn din,
                                                       const uint64_t* __restrict__ rg, uint64_t* __restrict__ rs,
                                                       const uint64_t* __restrict__ GS, const uint8_t* __restrict__ tflag,
                                                       const uint32_t* __restrict__ gfx_in,
                                                       const DevScalars* sc, FilterConst fc, int par)
{
    PDL_ENTER();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    RdSmem& S = *reinterpret_cast<RdSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    const RsConst rc = make_rsconst(sc, fc.nu, fc.force_exact != 0);
    out.s += fc.lo_cap - scrd(sc->o_base[par ^ 1]);
    if (rc.W == 0 && fc.world == 1) {   // empty world (A-26)
        for (uint32_t i = blockIdx.x * blockDim.x + tid; i < fc.nu; i += gridDim.x * blockDim.x)
            out.s[i] = make_float4(kSentinelPos, kSentinelPos, 0.0f, 0.0f);
    }
    const uint32_t n = tile_count(sc, par, base);
    if (n == 0 || !tflag[t]) return;                          // tiles without Doppler runs: k_resample_tiles
    const uint32_t nd = tp.nd[t];
    const uint32_t pbase = fc.lo_cap - scrd(sc->n_lo) + base;
    const RunInfo* __restrict__ runs = tp.run + base;
    const uint64_t Ppre = scrd(sc->Ppre);
    for (uint32_t w = tid; w < kSortTile / 32; w += 256) S.wrun[w] = 0u;
    __syncthreads();
    for (uint32_t r = tid; r < nd; r += 256) {             // run starts; weighted runs (parallel gathers)
        S.first[r] = tp.first[base + r];
        if (tp.key[base + r] < fc.C && GS[runs[r].li & ~kRunDirect] > 0) atomicOr(&S.wrun[r >> 5], 1u << (r & 31u));
    }
    if (tid == 0) S.first[nd] = (uint16_t)n;
    __syncthreads();
    auto weighted = [&](uint32_t r) { return ((S.wrun[r >> 5] >> (r & 31u)) & 1u) != 0u; };
    const uint32_t p0 = tid * kRdItems;
    const uint32_t p1 = min(p0 + kRdItems, n);

    // pass 1: gfx of the owned positions (k_dopp_runs wrote them in sorted order), thread total, block
    // prefix; run starts -> rs[run]
    uint32_t gf[kRdItems];
    uint64_t tsum = 0;
#pragma unroll
    for (int h = 0; h < kRdItems / 4; ++h) {
        uint4 w = make_uint4(0u, 0u, 0u, 0u);
        if (p0 + 4 * h < n) w = reinterpret_cast<const uint4*>(gfx_in + base + p0)[h];   // past n: masked below
        gf[4 * h] = p0 + 4 * h < p1 ? w.x : 0u;
        gf[4 * h + 1] = p0 + 4 * h + 1 < p1 ? w.y : 0u;
        gf[4 * h + 2] = p0 + 4 * h + 2 < p1 ? w.z : 0u;
        gf[4 * h + 3] = p0 + 4 * h + 3 < p1 ? w.w : 0u;
    }
#pragma unroll
    for (int u = 0; u < kRdItems; ++u) tsum += gf[u];
    uint64_t tot;
    const uint64_t tb = block_excl_scan<uint64_t, 8>(tsum, S.scan, tot);
    {
        uint64_t x = tb;
        uint32_t j = p0 < n ? run_of(S.first, nd, p0) : 0u;
        for (int u = 0; u < kRdItems; ++u) {
            const uint32_t p = p0 + u;
            if (p >= p1) break;
            while (S.first[j + 1] <= p) ++j;
            if (S.first[j] == p) rs[base + j] = x;            // block prefix at the run's first member
            x += gf[u];
        }
    }
    __syncthreads();                                          // rs[] visible to the block

    // pass 2: Q_j, Q_{j+1} -> outputs [F(P + Q_j), F(P + Q_{j+1})); velocity sums per run segment
    if (p0 < n) {
        uint32_t j = run_of(S.first, nd, p0);
        uint32_t first = S.first[j], end = S.first[j + 1];
        double acc[5] = {0, 0, 0, 0, 0};
        bool first_seg = true;
        uint64_t x = tb;
        auto load_run = [&](RunQ& q, uint32_t& key, uint64_t& Rp, uint32_t& nm, uint64_t& gsc, float& pa) {
            gsc = 0;
            key = fc.C;
            if (weighted(j)) {                                // (other runs: k_resample_tiles)
                key = tp.key[base + j];
                q = run_q(runs[j], L, Ppre);
                Rp = L.Rp[q.li]; nm = L.n[q.li]; gsc = GS[q.li];
                pa = din.pA[key];
            }
        };
        RunQ q{};
        uint32_t key = 0, nm = 0;
        uint64_t Rp = 0, gsc = 0;
        float pa = 0.0f;
        load_run(q, key, Rp, nm, gsc, pa);
        auto flush = [&]() {
            MomPartial mp;
#pragma unroll
            for (int i = 0; i < 5; ++i) { mp.s[i] = acc[i]; acc[i] = 0.0; }
            if (key < fc.C && gsc > 0) {
                if (first >= p0 && end <= p0 + kRdItems) ppart[base + j] = mp;   // run inside this thread
                else if (first_seg) S.pa[tid] = mp;
                else S.pb[tid] = mp;
            }
            first_seg = false;
        };
        uint64_t Qc = 0;                                      // Q_{j+1} / F(P + Q_{j+1}) of the previous member
        uint32_t Fc = 0;                                      // of the same run: the next member's Q_j / F
        bool have = false;
        for (int u = 0; u < kRdItems; ++u) {
            const uint32_t p = p0 + u;
            if (p >= p1) break;
            if (p >= end) {
                flush();
                ++j; first = end; end = S.first[j + 1];
                load_run(q, key, Rp, nm, gsc, pa);
                have = false;
            }
            const uint64_t xp = x;
            x += gf[u];
            if (key >= fc.C || gsc == 0) continue;            // outside the grid / no weights: k_resample_tiles
            const uint32_t mr = q.pre + (p - first);
            uint64_t Q0, Q1;
            if (gsc > 0) {
                const uint64_t g0 = rg[base + j] + (xp - rs[base + j]);
                Q0 = have ? Qc : doppler_Q(Rp, pa, g0, gsc, mr, nm);
                Q1 = doppler_Q(Rp, pa, g0 + gf[u], gsc, mr + 1, nm);
            } else {
                Q0 = (uint64_t)mr * q.bp + min(mr, q.rpm);
                Q1 = (uint64_t)(mr + 1) * q.bp + min(mr + 1, q.rpm);
            }
            const float2 XY = pxy[pbase + p], VV = pv[pbase + p];   // sorted order
            const float4 X = make_float4(XY.x, XY.y, VV.x, VV.y);
            if (rc.W) {
                const uint32_t F0 = have ? Fc : fcount(q.P + Q0, rc), F1 = fcount(q.P + Q1, rc);
                DOG_ASSERT(F0 <= F1 && F1 <= fc.nu);
                Fc = F1;
                for (uint32_t o = F0; o < F1; ++o) out.s[o] = X;
            }
            Qc = Q1;
            have = true;
            const double w = gsc > 0 ? (double)(Q1 - Q0) : 1.0;
            const double a = (double)X.z, b = (double)X.w;
            acc[0] += w * a; acc[1] += w * b; acc[2] += w * a * a; acc[3] += w * b * b; acc[4] += w * a * b;
        }
        flush();
    }
    __syncthreads();
    // spanning runs: the segments over threads tf..tl, combined by one warp per run (fixed lane tree:
    // deterministic) -> ppart
    const int warp = tid >> 5, lane = tid & 31;
    for (uint32_t r = warp; r < nd; r += 8) {
        const uint32_t f = S.first[r], e = S.first[r + 1];
        const uint32_t tf = f / kRdItems, tl = (e - 1) / kRdItems;
        if (tf == tl || !weighted(r)) continue;             // weighted runs over several threads only
        double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (uint32_t u = tf + 1 + lane; u <= tl; u += 32)
#pragma unroll
            for (int i = 0; i < 5; ++i) s5[i] += S.pa[u].s[i];
#pragma unroll
        for (int d = 16; d; d >>= 1)
#pragma unroll
            for (int i = 0; i < 5; ++i) s5[i] += __shfl_xor_sync(0xffffffffu, s5[i], d);
        if (lane == 0) {
            const MomPartial& m0 = (f > tf * kRdItems) ? S.pb[tf] : S.pa[tf];
            MomPartial mp;
#pragma unroll
            for (int i = 0; i < 5; ++i) mp.s[i] = m0.s[i] + s5[i];
            ppart[base + r] = mp;
        }
    }
}

}  // namespace dog
