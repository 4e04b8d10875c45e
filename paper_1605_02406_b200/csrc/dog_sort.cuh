// dog_sort.cuh -- Alg. 2: particle-to-cell assignment by a stable key sort, B200 style.
//
// The paper sorts the whole particle array by cell index (Thrust) and takes first/last indices per
// cell.  What the rest of the cycle needs from that sort is, for every particle, its cell and its
// stable rank among the particles of that cell (A-6: ties by input index).  Because the input is the
// previous resampling output -- already ordered by source cell -- and particles move a few cells per
// step, every 4096-particle tile holds few distinct cells.  So:
//   k_predict_sort : per tile, predict (Alg. 1) fused with a stable LSD radix sort of the tile's keys in
//                 shared memory (only the digits the tile's key range needs), runs of equal keys ->
//                 "pairs" (tile, cell, count, first local position), the local permutation, and per-cell
//                 counts n_c / pair counts.
//   k_pair_fill : each pair appends itself to its cell's pair list (position by atomic, unordered).
//   k_pair_sort : per active cell, its pair list sorted by tile (keys are unique: one run per tile per
//                 cell) and the exclusive prefix of the counts = the rank of each run's first particle
//                 among the cell's particles in input order.
// The global order (cell, input index) of the paper's sort is thereby fully determined without moving
// any particle: a particle's cell-sorted slot is start_c + pre(tile, run) + (position within the run).
#pragma once
#include <cstddef>
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_fcount.cuh"
#include "dog_kernels.cuh"
#include "dog_rng.cuh"

namespace dog {

#ifndef MO_DIRECT
#define MO_DIRECT 32
#endif
constexpr uint32_t kMoDirect = MO_DIRECT;   // long-list (run-heavy) cycles: cells with at most this many particles are
                                     // summed directly by k_moments<true> (resample skips their run sums)

// What the resampling kernels need of a run beyond its cell (written by k_pair_sort): 8 bytes per run --
// in the run-heavy regime of the exact filter (~1 member per run) the per-run record is a particle-sized
// stream, so the cell's own parameters are gathered from the list (consecutive runs of a tile belong to
// consecutive list entries: coalesced) instead of being copied into every run.
struct RunInfo {
    uint32_t pre;           // rank of the run's first particle among the cell's particles
    uint32_t li;            // the cell's active-list entry | kRunDirect
};
constexpr uint32_t kRunDirect = 0x80000000u;   // k_moments<true> sums the cell's velocities itself (<= kMoDirect
                                               // members): no run sums needed (list entries are < 2^31)

// A run with its cell's resampling parameters
struct RunQ {
    uint64_t P;             // joint-CDF prefix of the cell (A-25), including the shards below
    uint64_t bp;            // R_p / n_c of the cell (even split, A-23)
    uint32_t rpm;           // R_p mod n_c
    uint32_t pre;           // rank of the run's first particle among the cell's particles
    uint32_t li;            // the cell's active-list entry
    bool direct;
};
__device__ __forceinline__ RunQ run_q(RunInfo r, const CellList& L, uint64_t Ppre)
{
    RunQ q;
    q.li = r.li & ~kRunDirect;
    q.direct = (r.li & kRunDirect) != 0u;
    q.pre = r.pre;
    q.P = Ppre + L.P[q.li];
    q.bp = L.bp[q.li];
    q.rpm = L.rp[q.li];
    return q;
}

struct TilePairs {          // per tile t: entries [t*4096, t*4096 + nd[t])
    uint32_t* key;          // cell key of the run (C = outside the grid)
    uint16_t* first;        // first local sorted position of the run
    uint16_t* cnt;          // particles in the run (1..4096, stored as cnt-1)
    RunInfo* run;           // per-run resampling parameters                           (k_pair_sort)
    uint32_t* nd;           // [tiles] runs of the tile
};

// ------------------------------------------------------------------------------------------------
// Alg. 1 + the tile-local part of Alg. 2, fused: one block per 4096-particle tile predicts its particles
// (one Philox4x32-10 draw and two Box-Muller pairs each, A-1/A-2/A-20), keeps their cell keys in
// shared memory, sorts them stably (LSD radix over the bits of key - kmin the tile needs; 8-bit
// digits; ranks from match_any + per-warp running counters, so equal keys keep input order), and
// emits the runs of equal keys, the local permutation and per-cell counts.  Keys never touch HBM
// (debug builds write them for the KEY dump).
// ------------------------------------------------------------------------------------------------
constexpr int kPsThreads = 256, kPsWarps = kPsThreads / 32, kPsRows = kSortTile / kPsThreads;   // 16

// Sort records are packed (field << 12 | local index) in one u32 (a tile holds 4096 = 2^12 particles):
// one word moves per element and pass.  A remapped key of <= 20 bits is the field itself (the usual
// case); wider keys (a tile spread over > 2^20 cells of its bounding box) are sorted in two stable
// phases -- low 20 bits, then the high bits -- with the full keys kept in global scratch (kscr).
constexpr int kPkIdx = 12, kPkField = 32 - kPkIdx;   // 20-bit field
struct PsSmem {
    uint32_t k[2][kSortTile];          // packed records, ping-pong (k[0] holds the raw keys first)
    uint16_t rank[kSortTile];          // rank of each element among its warp's equal digits
    uint32_t hist[kPsWarps][256];      // per-warp digit counters -> scatter offsets
    uint32_t scan[kPsWarps + 1];
    uint32_t mn[kPsWarps], mx[kPsWarps];
};
constexpr size_t kPsSmemBytes = sizeof(PsSmem);
static_assert(offsetof(PsSmem, hist) == offsetof(PsSmem, rank) + kSortTile * 2 && sizeof(PsSmem::hist) == kSortTile * 2,
              "rank + hist form one 16 KB staging buffer");

// One particle of Alg. 1: p' = p + T v + xi_p with the OLD velocity (Eq. 14, A-2); v' = v + xi_v.  The
// four normals come from one Philox4x32-10 draw keyed by the particle's GLOBAL index (A-20), so a band
// context predicts exactly what a whole-grid context predicts for the same particle.
__device__ __forceinline__ float4 predict_one(float4 X, uint64_t gidx, const FilterConst& fc, const StepArgs& a)
{
    const Philox4 r = draw(fc.seed, (uint32_t)gidx, a.k, STAGE_PREDICT);
    float n0, n1, n2, n3;
    box_muller2(r.r0, r.r1, r.r2, r.r3, n0, n1, n2, n3);   // == box_muller(r0, r1), box_muller(r2, r3)
    const float xn = __fmaf_rn(a.s_p, n0, __fmaf_rn(X.z, a.Tc, X.x));
    const float yn = __fmaf_rn(a.s_p, n1, __fmaf_rn(X.w, a.Tc, X.y));
    return make_float4(xn, yn, __fmaf_rn(a.s_v, n2, X.z), __fmaf_rn(a.s_v, n3, X.w));
}

// Global cell key of a predicted particle: row * W + col inside the grid, Cg outside (A-4, A-5).
__device__ __forceinline__ uint32_t global_key(float4 P, const FilterConst& fc)
{
    const bool inside = (P.x >= 0.0f) && (P.x < (float)fc.W) && (P.y >= 0.0f) && (P.y < (float)fc.H);
    return inside ? (uint32_t)__float2int_rz(P.y) * (uint32_t)fc.W + (uint32_t)__float2int_rz(P.x) : fc.Cg;
}

// Context-local key: the cell within this context's band, C for anything outside it.
__device__ __forceinline__ uint32_t local_key(uint32_t kg, const FilterConst& fc)
{
    return (kg >= fc.c_off && kg - fc.c_off < fc.C) ? kg - fc.c_off : fc.C;
}

// Tiles cover the local particle array [s0, s0 + n_loc), s0 = lo_cap - n_lo (DevScalars).  kPredict:
// whole-grid context, predict + sort fused (own particles only).  !kPredict: band context, the tile's
// particles were predicted by k_predict_band (own) or by the neighbour shard (migrants): keys only.
// Warp w owns positions [512 w, 512 w + 512) as 16 rows of 32 lanes (position = 512 w + 32 i + lane).
//
// The predicted state leaves the kernel IN SORTED ORDER, as two halves: pxy[s0 + tb + p] = (x, y) and
// pv[s0 + tb + p] = (vx, vy) of the particle at sorted position p of the tile (staged through shared
// memory after the sort: every later pass reads it coalesced, in cell order).  kPredict writes the
// predicted halves in input order first and permutes them in place; !kPredict reads the band's records
// (pst, input order) and writes the halves.  pst (kPredict) and lperm are debug outputs (may be null).
template <bool kPredict>
__global__ __launch_bounds__(kPsThreads) void k_predict_sort(
    const float4* __restrict__ st, float4* __restrict__ pst, float2* __restrict__ pxy, float2* __restrict__ pv,
    uint32_t* __restrict__ keys_dbg, uint16_t* __restrict__ lperm, TilePairs tp, uint32_t* __restrict__ counts,
    uint32_t* __restrict__ npairs, DevScalars* sc, FilterConst fc, StepArgs a, uint32_t* __restrict__ kscr)
{
    PDL_ENTER();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    PsSmem& S = *reinterpret_cast<PsSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int par = (int)(a.k & 1);
    const uint32_t n_lo = scrd(sc->n_lo), n_own = scrd(sc->n_own[par]), n_loc = n_lo + n_own + scrd(sc->n_hi);
    const uint64_t o_base = scrd(sc->o_base[par]);
    const uint32_t s0 = fc.lo_cap - n_lo;
    const uint32_t tb = blockIdx.x * kSortTile;                // this tile's slot in the per-tile arrays
    const uint32_t base = s0 + tb;                             // its first particle
    const uint32_t n = n_loc > tb ? min((uint32_t)kSortTile, n_loc - tb) : 0u;
    if (kPredict) {
        const float w_bar = scrd(sc->w_bar);
        const float w_pred = __fmul_rn(fc.p_s, w_bar);      // Eq. 39 (A-3): one scalar
        if (blockIdx.x == 0 && tid == 0) { sc->w_pred = w_pred; sc->A_acc = 0ull; }
    }

    PHASE_BEGIN();
    // ---- predict (Alg. 1) or load: position p = local index (input order).  The sort key is the
    //      (row, col) of the particle's cell, packed, remapped below onto the tile's bounding box of
    //      cells: (row - rmin) * span + (col - cmin) preserves the cell order and usually needs 8-10 bits
    //      (one or two radix passes instead of the 13+ bits of the cell index itself).
    constexpr uint32_t kOut = 0xFFFFFFFEu;                  // outside the context's band (or the grid)
    uint32_t rmin = 0xFFFFu, rmax = 0u, cmin = 0xFFFFu, cmax = 0u, anyout = 0u;
#pragma unroll 4
    for (int i = 0; i < kPsRows; ++i) {
        const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
        uint32_t key = 0xFFFFFFFFu;
        if (p < n) {
            const uint32_t g = base + p;
            float4 P;
            if (kPredict) {
                P = predict_one(st[g], o_base + (g - fc.lo_cap), fc, a);
                pxy[g] = make_float2(P.x, P.y);
                pv[g] = make_float2(P.z, P.w);
                if (pst) pst[g] = P;                        // debug: the predicted state in input order
            } else {
                P = pst[g];
            }
            const uint32_t kg = global_key(P, fc);
            if (keys_dbg) keys_dbg[g] = kg;
            if (local_key(kg, fc) < fc.C) {
                const uint32_t row = (uint32_t)__float2int_rz(P.y), col = (uint32_t)__float2int_rz(P.x);
                key = (row << 16) | col;
                rmin = min(rmin, row); rmax = max(rmax, row); cmin = min(cmin, col); cmax = max(cmax, col);
            } else {
                key = kOut;
                anyout = 1u;
            }
        }
        S.k[0][p] = key;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, off));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
        cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, off));
        cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
        anyout |= __shfl_xor_sync(0xffffffffu, anyout, off);
    }
    if (lane == 0) { S.mn[warp] = (rmin << 16) | cmin; S.mx[warp] = (rmax << 16) | cmax; S.rank[warp] = (uint16_t)anyout; }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kPsWarps; ++w) {
        rmin = min(rmin, S.mn[w] >> 16); cmin = min(cmin, S.mn[w] & 0xFFFFu);
        rmax = max(rmax, S.mx[w] >> 16); cmax = max(cmax, S.mx[w] & 0xFFFFu);
        anyout |= S.rank[w];
    }
    if (n == 0) {                                           // beyond the particles of this cycle
        if (tid == 0) tp.nd[blockIdx.x] = 0u;
        return;
    }
    PHASE_MARK(8);
    const bool anyin = rmin <= rmax;
    const uint32_t span = anyin ? cmax - cmin + 1u : 1u, rows = anyin ? rmax - rmin + 1u : 0u;
    const uint32_t kout = rows * span;                      // the remapped key of "outside": after every cell
    __syncthreads();                                        // S.rank reused below
    const uint32_t range = anyout ? kout : (anyin ? kout - 1u : 0u);
    const int bits = range ? 32 - __clz(range) : 0;
    const bool wide = bits > kPkField;                      // rare: two-phase sort, keys in kscr
#pragma unroll 4
    for (int i = 0; i < kPsRows; ++i) {                     // remap in place, pack (field << 12 | p)
        const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
        const uint32_t key = S.k[0][p];
        if (p < n) {
            const uint32_t rk = key == kOut ? kout : ((key >> 16) - rmin) * span + ((key & 0xFFFFu) - cmin);
            if (wide) kscr[tb + p] = rk;
            S.k[0][p] = ((wide ? (rk & ((1u << kPkField) - 1u)) : rk) << kPkIdx) | p;
        } else {
            S.k[0][p] = 0xFFFFFFFFu;                         // stays last
        }
    }
    __syncthreads();
#ifdef DOG_TIMING
    if (tid == 0) { atomicAdd(&g_phase_ns[30], (unsigned long long)((bits + 7) / 8)); atomicAdd(&g_phase_ns[31], 1ull); }
#endif

    // ---- stable LSD radix passes over the packed field (positions >= n stay at the end)
    int cur = 0;
    auto passes = [&](int nbits) {
        for (int shift = 0; shift < nbits; shift += 8, cur ^= 1) {
            for (int i = tid; i < kPsWarps * 256; i += kPsThreads) (&S.hist[0][0])[i] = 0;
            __syncthreads();
#pragma unroll 4
            for (int i = 0; i < kPsRows; ++i) {              // count + per-warp ranks
                const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
                const uint32_t w = S.k[cur][p];
                const uint32_t dig = p < n ? (w >> (kPkIdx + shift)) & 255u : 256u;
                const uint32_t peers = __match_any_sync(0xffffffffu, dig);
                uint32_t prev = 0;
                if (dig < 256u) prev = S.hist[warp][dig];
                __syncwarp();
                if (dig < 256u && (peers & lt) == 0) S.hist[warp][dig] = prev + __popc(peers);
                __syncwarp();
                S.rank[p] = (uint16_t)(prev + __popc(peers & lt));
            }
            __syncthreads();
            {   // digit d = tid: offsets over (digit, warp) in that order
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < kPsWarps; ++w) { const uint32_t c = S.hist[w][tid]; S.hist[w][tid] = run; run += c; }
                uint32_t tot;
                const uint32_t ds = block_excl_scan<uint32_t, kPsWarps>(run, S.scan, tot);
#pragma unroll
                for (int w = 0; w < kPsWarps; ++w) S.hist[w][tid] += ds;
            }
            __syncthreads();
#pragma unroll 4
            for (int i = 0; i < kPsRows; ++i) {              // scatter
                const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
                if (p >= n) continue;
                const uint32_t w = S.k[cur][p];
                const uint32_t dig = (w >> (kPkIdx + shift)) & 255u;
                S.k[cur ^ 1][S.hist[warp][dig] + S.rank[p]] = w;
            }
            __syncthreads();
        }
    };
    if (!wide) {
        passes(bits);
    } else {
        passes(kPkField);                                   // low 20 bits
        for (int i = 0; i < kPsRows; ++i) {                 // repack with the high bits
            const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
            if (p < n) {
                const uint32_t w = S.k[cur][p], q = w & ((1u << kPkIdx) - 1u);
                S.k[cur][p] = ((kscr[tb + q] >> kPkField) << kPkIdx) | q;
            }
        }
        __syncthreads();
        passes(bits - kPkField);
    }
    PHASE_MARK(9);
    const uint32_t* sw = S.k[cur];                          // sorted packed records
    auto skey = [&](uint32_t p) -> uint32_t {               // remapped key of sorted position p
        const uint32_t w = sw[p];
        return wide ? kscr[tb + (w & ((1u << kPkIdx) - 1u))] : (w >> kPkIdx);
    };

    // ---- runs of equal keys (warp rows -> heads in position order)
    uint32_t hb[kPsRows];
    uint32_t wc = 0;
#pragma unroll
    for (int i = 0; i < kPsRows; ++i) {
        const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
        const bool head = p < n && (p == 0 || skey(p) != skey(p - 1));
        hb[i] = __ballot_sync(0xffffffffu, head);
        wc += __popc(hb[i]);
    }
    uint32_t nd;
    uint32_t j = block_excl_scan<uint32_t, kPsWarps>(lane == 0 ? wc : 0u, S.scan, nd);
    j = __shfl_sync(0xffffffffu, j, 0);
    uint16_t* s_start = S.rank;                             // reuse: run starts (nd <= n)
#pragma unroll
    for (int i = 0; i < kPsRows; ++i) {
        const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
        if ((hb[i] >> lane) & 1u) s_start[j + __popc(hb[i] & lt)] = (uint16_t)p;
        j += __popc(hb[i]);
    }
    __syncthreads();
    for (uint32_t r = tid; r < nd; r += kPsThreads) {
        const uint32_t f = s_start[r], e = r + 1 < nd ? (uint32_t)s_start[r + 1] : n, c = e - f;
        const uint32_t kr = skey(f);                       // remapped key -> the context's cell index
        const uint32_t key = kr >= kout ? fc.C
                           : (rmin + kr / span - fc.row0) * (uint32_t)fc.W + cmin + kr % span;
        tp.key[tb + r] = key;
        tp.first[tb + r] = (uint16_t)f;
        tp.cnt[tb + r] = (uint16_t)(c - 1);
        if (key < fc.C) {
            atomicAdd(&counts[key], c);
            atomicAdd(&npairs[key], 1u);
        }
    }
    if (tid == 0) tp.nd[blockIdx.x] = nd;
    PHASE_MARK(10);
    // ---- local permutation (sorted position -> local input index): debug dumps only
    if (lperm)
        for (uint32_t q = tid; 2 * q < n; q += kPsThreads) {
            const uint32_t p = 2 * q;
            const uint32_t v0 = sw[p] & ((1u << kPkIdx) - 1u), v1 = sw[p + 1] & ((1u << kPkIdx) - 1u);
            reinterpret_cast<uint32_t*>(lperm + tb)[q] = v0 | (v1 << 16);
        }
    __syncthreads();                                        // s_start (S.rank) is free again
    // ---- the predicted state in sorted order: each half staged through shared memory in input order
    //      (coalesced reads, conflict-free stores), then gathered by sorted position through the
    //      sorted records (sorted position -> local index) and written back coalesced
    float* st0 = reinterpret_cast<float*>(S.k[cur ^ 1]);                // 16 KB
    float* st1 = reinterpret_cast<float*>(S.rank);                      // rank + hist: 16 KB
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        float2* dst = h ? pv : pxy;
#pragma unroll 4
        for (int i = 0; i < kPsRows; ++i) {
            const uint32_t q = warp * (kPsRows * 32) + i * 32 + lane;
            if (q < n) {
                float2 v;
                if (kPredict) {
                    v = dst[base + q];
                } else {
                    const float4 P = pst[base + q];
                    v = h ? make_float2(P.z, P.w) : make_float2(P.x, P.y);
                }
                st0[q] = v.x;
                st1[q] = v.y;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int i = 0; i < kPsRows; ++i) {
            const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
            if (p < n) {
                const uint32_t q = sw[p] & ((1u << kPkIdx) - 1u);
                dst[base + p] = make_float2(st0[q], st1[q]);
            }
        }
        __syncthreads();
    }
    PHASE_MARK(11);
}

// ------------------------------------------------------------------------------------------------
// Row-band contexts: Alg. 1 for the own particles, then the particles whose
// new cell lies in another band are packed, in input (= global index) order, into four buckets: for the
// band below, the band above, and the bands further below / above (owner-bucketed: any displacement
// reaches its band, nothing is dropped).  Their slots in the local array keep them with a key outside
// the band, so the local sort leaves them out (like particles outside the grid).
// ------------------------------------------------------------------------------------------------
constexpr int kMigDirs = 4;   // 0 below, 1 above, 2 further below, 3 further above
struct Migrants {
    float4* scr[kMigDirs];     // per tile, compacted: [tile * 4096 + k]
    uint32_t* cnt[kMigDirs];   // per tile
    float4* send[kMigDirs];    // packed for the receivers (capacity cap each)
    uint32_t cap;
};

__global__ __launch_bounds__(kPsThreads) void k_predict_band(const float4* __restrict__ st, float4* __restrict__ pst,
                                                             Migrants mg, DevScalars* sc, FilterConst fc,
                                                             StepArgs a)
{
    PDL_ENTER();
    __shared__ uint32_t s_w[kMigDirs][kPsWarps + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int par = (int)(a.k & 1);
    const uint32_t n_own = scrd(sc->n_own[par]);
    const uint64_t o_base = scrd(sc->o_base[par]);
    const uint32_t tb = blockIdx.x * kSortTile;
    const uint32_t n = n_own > tb ? min((uint32_t)kSortTile, n_own - tb) : 0u;
    if (blockIdx.x == 0 && tid == 0) {
        sc->w_pred = __fmul_rn(fc.p_s, scrd(sc->w_bar));         // Eq. 39 (A-3)
        sc->A_acc = 0ull;
    }
    float4 P[kPsRows];
    uint32_t dir[kPsRows];                                  // kMigDirs: stays (or leaves the grid)
    uint32_t wc[kMigDirs] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < kPsRows; ++i) {
        const uint32_t p = warp * (kPsRows * 32) + i * 32 + lane;
        dir[i] = kMigDirs;
        if (p < n) {
            const uint32_t q = fc.lo_cap + tb + p;
            P[i] = predict_one(st[q], o_base + tb + p, fc, a);
            pst[q] = P[i];
            const uint32_t kg = global_key(P[i], fc);
            if (kg < fc.Cg && kg < fc.c_off) dir[i] = kg >= fc.c_lo ? 0u : 2u;
            else if (kg < fc.Cg && kg - fc.c_off >= fc.C) dir[i] = kg < fc.c_hi ? 1u : 3u;
        }
#pragma unroll
        for (int d = 0; d < kMigDirs; ++d) wc[d] += __popc(__ballot_sync(0xffffffffu, dir[i] == (uint32_t)d));
    }
    if (lane == 0)
#pragma unroll
        for (int d = 0; d < kMigDirs; ++d) s_w[d][warp] = wc[d];
    __syncthreads();
    uint32_t off[kMigDirs] = {0, 0, 0, 0}, tot[kMigDirs] = {0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < kPsWarps; ++w)
#pragma unroll
        for (int d = 0; d < kMigDirs; ++d) { if (w < warp) off[d] += s_w[d][w]; tot[d] += s_w[d][w]; }
#pragma unroll
    for (int i = 0; i < kPsRows; ++i) {
        if (__ballot_sync(0xffffffffu, dir[i] < (uint32_t)kMigDirs) == 0u) continue;   // ~99 %: nobody leaves
#pragma unroll
        for (int d = 0; d < kMigDirs; ++d) {
            const uint32_t b = __ballot_sync(0xffffffffu, dir[i] == (uint32_t)d);
            if (dir[i] == (uint32_t)d) mg.scr[d][tb + off[d] + __popc(b & lt)] = P[i];
            off[d] += __popc(b);
        }
    }
    if (tid < kMigDirs) mg.cnt[tid][blockIdx.x] = tot[tid];
}

// One block: exclusive prefix of the per-tile migrant counts of each bucket, then the packed send
// buffers (input order, one warp per tile copying lane-strided); totals go to DevScalars (read by the
// receivers' k_gather_migrants, or by the host to size a transport).  A bucket beyond the capacity is
// truncated and flagged (mig_over): the cycle then cannot complete exactly and the host reports it.
__global__ __launch_bounds__(1024) void k_pack_migrants(Migrants mg, uint32_t tiles, DevScalars* sc)
{
    PDL_ENTER();
    __shared__ uint32_t s_run;
    __shared__ uint32_t s_w[33];
    __shared__ uint32_t s_off[1024], s_cnt[1024];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = 0; d < kMigDirs; ++d) {
        if (tid == 0) s_run = 0u;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < tiles; t0 += 1024) {
            const uint32_t t = t0 + tid;
            const uint32_t c = t < tiles ? mg.cnt[d][t] : 0u;
            const uint32_t inc = warp_incl_scan(c, lane);
            if (lane == 31) s_w[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                const uint32_t v = s_w[lane];
                const uint32_t vi = warp_incl_scan(v, lane);
                s_w[lane] = vi - v;
                if (lane == 31) s_w[32] = vi;
            }
            __syncthreads();
            s_off[tid] = s_run + s_w[warp] + inc - c;
            s_cnt[tid] = c;
            __syncthreads();
            const uint32_t nt = min(1024u, tiles - t0);
            for (uint32_t u = warp; u < nt; u += 32) {     // warp per tile (migrants are ~1 %)
                const uint32_t cu = s_cnt[u], dst0 = s_off[u];
                const float4* src = mg.scr[d] + (size_t)(t0 + u) * kSortTile;
                for (uint32_t k = lane; k < cu; k += 32)
                    if (dst0 + k < mg.cap) mg.send[d][dst0 + k] = src[k];
            }
            __syncthreads();
            if (tid == 0) s_run += s_w[32];
            __syncthreads();
        }
        if (tid == 0) {
            sc->mig_cnt[d] = min(s_run, mg.cap);
            if (s_run > mg.cap) sc->mig_over = 1u;
        }
    }
}

// Where a band's migrants come from (device pointers readable from the receiver: its own memory, a
// peer GPU's over NVLink, or a transport's receive buffer), each bucket with its device count.
constexpr int kMaxBands = 16;
struct MigSrc {
    const float4* rec;
    const uint32_t* cnt;
};
struct MigGather {
    MigSrc lo_near, hi_near;        // bucket 1 of band r-1 / bucket 0 of band r+1 (all of it is for r)
    MigSrc lo_far[kMaxBands];       // bucket 3 of bands 0 .. r-2, in band order (filtered by row)
    MigSrc hi_far[kMaxBands];       // bucket 2 of bands r+2 .. world-1, in band order (filtered by row)
    int n_lo_far, n_hi_far;
};

// Receiver: builds [from below | own | from above] in global index order around the own particles
// (pst[lo_cap .. lo_cap + n_own)): from below = the far records of bands 0 .. r-2 that land in this band,
// then all of band r-1's near bucket, ending at lo_cap; from above = band r+1's near bucket, then the
// far records of bands r+2 .. that land here.  Blocks 1.. copy the near buckets (contiguous); block 0
// compacts the far buckets (rare) with block scans and publishes n_lo / n_hi.  A receive beyond the
// capacity copies nothing and raises mig_over.
__global__ __launch_bounds__(1024) void k_gather_migrants(MigGather g, float4* __restrict__ pst,
                                                          DevScalars* sc, FilterConst fc,
                                                          uint32_t own_hi_cap, int par)
{
    PDL_ENTER();
    __shared__ uint32_t s_w[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n_own = scrd(sc->n_own[par]);
    const uint32_t hi_room = own_hi_cap - n_own;              // slots after the own particles
    const uint32_t nlo = g.lo_near.rec ? __ldcg(g.lo_near.cnt) : 0u;   // the senders' counts: from L2
    const uint32_t nhi = g.hi_near.rec ? __ldcg(g.hi_near.cnt) : 0u;
    float4* const lo_end = pst + fc.lo_cap;
    float4* const hi_beg = pst + fc.lo_cap + n_own;
    if (blockIdx.x > 0) {
        const uint32_t nb = gridDim.x - 1, b = blockIdx.x - 1;
        if (nlo <= fc.lo_cap)
            for (uint32_t i = b * 1024 + tid; i < nlo; i += nb * 1024) lo_end[(int64_t)i - nlo] = g.lo_near.rec[i];
        if (nhi <= hi_room)
            for (uint32_t i = b * 1024 + tid; i < nhi; i += nb * 1024) hi_beg[i] = g.hi_near.rec[i];
        return;
    }
    // block 0: far records landing in this band, stable compaction in band order
    auto in_band = [&](const float4& P) {
        const uint32_t kg = global_key(P, fc);
        return kg < fc.Cg && kg >= fc.c_off && kg - fc.c_off < fc.C;
    };
    auto block_excl = [&](uint32_t f, uint32_t& tot) -> uint32_t {
        const uint32_t b = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_w[warp] = __popc(b);
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = s_w[lane];
            const uint32_t vi = warp_incl_scan(v, lane);
            s_w[lane] = vi - v;
            if (lane == 31) s_w[32] = vi;
        }
        __syncthreads();
        const uint32_t r = s_w[warp] + __popc(b & ((1u << lane) - 1u));
        tot = s_w[32];
        __syncthreads();
        return r;
    };
    // pass 1: far records from below (their total places them before the near bucket)
    uint32_t flo = 0;
    for (int s = 0; s < g.n_lo_far; ++s) {
        const uint32_t n = __ldcg(g.lo_far[s].cnt);
        for (uint32_t i0 = 0; i0 < n; i0 += 1024) {
            const uint32_t i = i0 + tid;
            flo += (uint32_t)__syncthreads_count(i < n && in_band(g.lo_far[s].rec[i]));
        }
    }
    const bool lo_ok = nlo + flo <= fc.lo_cap;
    uint32_t pos = 0;
    for (int s = 0; s < g.n_lo_far && lo_ok; ++s) {
        const uint32_t n = __ldcg(g.lo_far[s].cnt);
        for (uint32_t i0 = 0; i0 < n; i0 += 1024) {
            const uint32_t i = i0 + tid;
            float4 P = make_float4(0.f, 0.f, 0.f, 0.f);
            const bool f = i < n && in_band(P = g.lo_far[s].rec[i]);
            uint32_t tot;
            const uint32_t r = block_excl(f, tot);
            if (f) lo_end[(int64_t)pos + r - (nlo + flo)] = P;
            pos += tot;
        }
    }
    uint32_t fhi = 0;
    const bool near_hi_ok = nhi <= hi_room;
    for (int s = 0; s < g.n_hi_far && near_hi_ok; ++s) {
        const uint32_t n = __ldcg(g.hi_far[s].cnt);
        for (uint32_t i0 = 0; i0 < n; i0 += 1024) {
            const uint32_t i = i0 + tid;
            float4 P = make_float4(0.f, 0.f, 0.f, 0.f);
            const bool f = i < n && in_band(P = g.hi_far[s].rec[i]);
            uint32_t tot;
            const uint32_t r = block_excl(f, tot);
            if (f && nhi + fhi + r < hi_room) hi_beg[nhi + fhi + r] = P;
            fhi += tot;
        }
    }
    if (tid == 0) {
        const bool hi_ok = nhi + fhi <= hi_room;
        sc->n_lo = lo_ok ? nlo + flo : 0u;
        sc->n_hi = hi_ok ? nhi + fhi : 0u;
        if (!lo_ok || !hi_ok) sc->mig_over = 1u;
    }
}

// Each pair appends itself (tile << 12 | run) to its cell's list (unordered; k_pair_sort orders it).
__global__ __launch_bounds__(256) void k_pair_fill(TilePairs tp, CellList L, const uint32_t* __restrict__ cell2list,
                                                   uint32_t* __restrict__ plist, uint32_t C)
{
    PDL_ENTER();
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    const uint32_t nd = tp.nd[t];
    for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x) {
        const uint32_t key = tp.key[base + r];
        if (key >= C) continue;
        const uint32_t li = cell2list ? cell2list[key] : key;    // (dense cycles: entry = cell)
        const uint32_t slot = atomicAdd(&L.pfill[li], 1u);
        DOG_ASSERT(slot < L.np[li]);
        plist[L.ps[li] + slot] = (t << 12) | r;
    }
}

// Per active cell: its pair list sorted by tile, then the exclusive prefix of the run counts in that
// order -> pre of every run, and the run's resampling parameters (RunInfo).  Groups of 8 lanes take one
// cell each (4 cells per warp, so neighbouring cells with long lists proceed in parallel); lists are
// staged in shared memory and sorted by rank-by-count (entries are distinct, lists are short).
constexpr int kPsGroup = 8, kPsBuf = 128;

// W_all: joint weight of every shard (band contexts, gathered after k_list_scan) or nullptr (whole grid).
// Block 0 also publishes the cycle's global totals: W over all shards, the joint prefix of the shards
// below, w_bar = W 2^-40 / nu (Eq. 57), and -- band contexts -- the next cycle's own particles: the
// global outputs [F(P'), F(P' + W_local)) (A-24).
// Doppler branch (NEXT-1; pA == nullptr otherwise): the per-run likelihood sums rg (k_dopp_runs) of a
// Doppler cell become, in the same tile-order walk, their exclusive prefixes within the cell; GS[li] =
// the cell's total (0: no Doppler weighting, A-35) and tflag marks the tiles holding such a cell's runs.
struct DopPS {
    const float* pA;
    uint64_t* rg;
    uint64_t* GS;
    uint8_t* tflag;
    uint32_t* gmax;   // the cells' likelihood maxima (k_dopp_g): cleared here for the next cycle (or nullptr)
};

constexpr int kPsSmall = 4;   // kBatch: cells with <= 4 runs handled by one lane (sorting network)
static_assert(kPsSmall == 4, "the sorting network below is for 4 entries");
template <bool kBatch>
__global__ __launch_bounds__(256) void k_pair_sort(TilePairs tp, CellList L, uint32_t* __restrict__ plist,
                                                   uint32_t* __restrict__ ptmp, const uint64_t* __restrict__ W_all,
                                                   DevScalars* sc, FilterConst fc, int par, DopPS dp)
{
    PDL_ENTER();
    __shared__ uint32_t s_buf[256 / kPsGroup][2][kPsBuf];
    const int lane = threadIdx.x & 31, gl = lane & (kPsGroup - 1), grp = threadIdx.x / kPsGroup;
    const uint32_t gmask = 0xFFu << (lane & ~(kPsGroup - 1));
    const uint32_t Lc = scrd(sc->Lc);
    uint64_t Ppre = 0, Wtot = scrd(sc->W);
    if (W_all) {
        Wtot = 0;
        for (uint32_t r = 0; r < fc.world; ++r) { if (r < fc.rank) Ppre += W_all[r]; Wtot += W_all[r]; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->Wtot = Wtot;
        sc->Ppre = Ppre;
        sc->w_bar = Wtot ? __double2float_rn(__ddiv_rn(__dmul_rn((double)Wtot, fc.fx_inv), (double)fc.nu)) : 0.0f;
        sc->nu_over_W = Wtot ? (double)fc.nu / (double)Wtot : 0.0;
        if (W_all) {
            RsConst r;
            r.exact = fc.force_exact != 0;
            r.W = Wtot; r.U = scrd(sc->U); r.nu = fc.nu;
            r.nu_over_W = Wtot ? (double)fc.nu / (double)Wtot : 0.0;
            r.U_frac = (double)r.U * 0x1p-32;
            r.UW = (u128)r.U * (u128)Wtot;
            const uint32_t f0 = Wtot ? fcount(Ppre, r) : 0u;
            const uint32_t f1 = Wtot ? fcount(Ppre + scrd(sc->W), r) : 0u;
            sc->o_base[par ^ 1] = f0;
            sc->n_own[par ^ 1] = f1 - f0;
        }
    }
    auto run_info = [&](uint32_t li) {
        RunInfo ri;
        ri.pre = 0u;
        ri.li = li | (kBatch && L.n[li] <= kMoDirect ? kRunDirect : 0u);
        return ri;
    };
    auto dop_single = [&](uint32_t li, uint32_t v) {     // a one-run cell: its prefix is 0, its total the run's
        if (!dp.pA) return;
        const uint32_t c = L.c[li];
        const bool dc = dp.pA[c] > 0.0f;
        if (dc && dp.gmax) dp.gmax[c] = 0u;
        const uint64_t gs = dc ? dp.rg[v] : 0ull;
        dp.rg[v] = 0ull;
        dp.GS[li] = gs;
        if (gs) dp.tflag[v >> 12] = 1;
    };
    auto single = [&](uint32_t li, uint32_t m = 1u) {     // one run: pre = 0
        uint32_t* pl = plist + L.ps[li];
        if constexpr (!kBatch) {
            tp.run[pl[0]] = run_info(li);
            dop_single(li, pl[0]);
            return;
        }
        if (m == 1u) {
            tp.run[pl[0]] = run_info(li);
            dop_single(li, pl[0]);
            return;
        }
        // kBatch (exact filter): 2..kPsSmall runs sorted by one lane in registers (a 4-element sorting
        // network; entries are distinct), then the exclusive prefix of their counts (and, likelihood
        // cells of the exact filter with a likelihood, of the runs' likelihood sums)
        uint32_t v[kPsSmall];
#pragma unroll
        for (int q = 0; q < kPsSmall; ++q) v[q] = (uint32_t)q < m ? pl[q] : 0xFFFFFFFFu;
        auto cs = [](uint32_t& x, uint32_t& y) { const uint32_t lo = min(x, y), hi = max(x, y); x = lo; y = hi; };
        cs(v[0], v[1]); cs(v[2], v[3]); cs(v[0], v[2]); cs(v[1], v[3]); cs(v[1], v[2]);
        RunInfo r2 = run_info(li);
        uint32_t carry = 0;
        const bool dcell = dp.pA && dp.pA[L.c[li]] > 0.0f;
        if (dcell && dp.gmax) dp.gmax[L.c[li]] = 0u;
        uint64_t gcarry = 0;
#pragma unroll
        for (int q = 0; q < kPsSmall; ++q) {
            if ((uint32_t)q < m) {
                r2.pre = carry;
                tp.run[v[q]] = r2;
                pl[q] = v[q];                                 // the cell's list, now in tile order
                carry += (uint32_t)tp.cnt[v[q]] + 1u;
                if (dcell) {
                    const uint64_t g = dp.rg[v[q]];
                    dp.rg[v[q]] = gcarry;
                    gcarry += g;
                }
            }
        }
        if (dp.pA) {
            dp.GS[li] = gcarry;
            if (gcarry)
#pragma unroll
                for (int q = 0; q < kPsSmall; ++q)
                    if ((uint32_t)q < m) dp.tflag[v[q] >> 12] = 1;
        }
    };
    for_run_entries<kBatch, kPsGroup, kBatch ? kPsSmall : 1>(L.np, Lc, [&](uint32_t li, uint32_t m) {
        const RunInfo ri = run_info(li);
        uint32_t* pl = plist + L.ps[li];
        if (m == 1) {                                 // (tile << 12 | run) is the run's slot index
            if (gl == 0) { tp.run[pl[0]] = ri; dop_single(li, pl[0]); }
            return;
        }
        const bool dcell = dp.pA && dp.pA[L.c[li]] > 0.0f;
        if (dcell && dp.gmax && gl == 0) dp.gmax[L.c[li]] = 0u;
        const bool sm = m <= (uint32_t)kPsBuf;
        uint32_t* src = sm ? s_buf[grp][0] : pl;
        uint32_t* tmp = sm ? s_buf[grp][1] : ptmp + L.ps[li];
        const uint32_t mr = (m + kPsGroup - 1) / kPsGroup * kPsGroup;   // group-uniform trip counts
        if (sm)
            for (uint32_t a = gl; a < m; a += kPsGroup) src[a] = pl[a];
        __syncwarp(gmask);
        // rank of each entry = number of smaller entries (entries are distinct)
        for (uint32_t a = gl; a < m; a += kPsGroup) {
            const uint32_t va = src[a];
            uint32_t rank = 0;
            for (uint32_t q = 0; q < m; ++q) rank += src[q] < va ? 1u : 0u;
            tmp[rank] = va;
        }
        __syncwarp(gmask);
        // exclusive prefix of counts (and, Doppler cells, of the runs' likelihood sums) in tile order
        uint32_t carry = 0;
        uint64_t gcarry = 0;
        for (uint32_t a0 = 0; a0 < mr; a0 += kPsGroup) {
            const uint32_t a = a0 + gl;
            uint32_t v = 0, c = 0;
            uint64_t g = 0;
            if (a < m) {
                v = tmp[a];
                c = (uint32_t)tp.cnt[v] + 1u;
                if (dcell) g = dp.rg[v];
            }
            uint32_t incl = c;
            uint64_t gincl = g;
#pragma unroll
            for (int d = 1; d < kPsGroup; d <<= 1) {
                const uint32_t o = __shfl_up_sync(gmask, incl, d, kPsGroup);
                const uint64_t go = __shfl_up_sync(gmask, gincl, d, kPsGroup);
                if (gl >= d) { incl += o; gincl += go; }
            }
            if (a < m) {
                RunInfo r2 = ri;
                r2.pre = carry + incl - c;
                tp.run[v] = r2;
                pl[a] = v;                   // the cell's list, now in tile order
                if (dp.pA) dp.rg[v] = gcarry + gincl - g;
            }
            carry += __shfl_sync(gmask, incl, kPsGroup - 1, kPsGroup);
            gcarry += __shfl_sync(gmask, gincl, kPsGroup - 1, kPsGroup);
        }
        if (dp.pA) {
            if (gl == 0) dp.GS[li] = gcarry;
            if (gcarry)
                for (uint32_t a = gl; a < m; a += kPsGroup) dp.tflag[pl[a] >> 12] = 1;
        }
        __syncwarp(gmask);
    }, single);
}

}  // namespace dog
