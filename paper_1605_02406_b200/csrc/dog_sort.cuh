// dog_sort.cuh -- Alg. 2: particle-to-cell assignment by a stable key sort, B200 style.
//
// The paper sorts the whole particle array by cell index (Thrust) and takes first/last indices per
// cell.  What the rest of the cycle needs from that sort is, for every particle, its cell and its
// stable rank among the particles of that cell (A-6: ties by input index).  Because the input is the
// previous resampling output -- already ordered by source cell -- and particles move a few cells per
// step, every 4096-particle tile holds few distinct cells.  So:
//   k_tilesort  : per tile, a stable LSD radix sort of the tile's keys in shared memory (only the
//                 digits the tile's key range needs), runs of equal keys -> "pairs" (tile, cell, count,
//                 first local position), the local permutation, and per-cell counts n_c / pair counts.
//   k_pair_fill : each pair appends itself to its cell's pair list (position by atomic, unordered).
//   k_pair_sort : per active cell, its pair list sorted by tile (keys are unique: one run per tile per
//                 cell) and the exclusive prefix of the counts = the rank of each run's first particle
//                 among the cell's particles in input order.
// The global order (cell, input index) of the paper's sort is thereby fully determined without moving
// any particle: a particle's cell-sorted slot is start_c + pre(tile, run) + (position within the run).
#pragma once
#include <cstdint>
#include "dog_cells.cuh"
#include "dog_common.cuh"
#include "dog_kernels.cuh"

namespace dog {

constexpr int kTsThreads = 256, kTsItems = 16, kTsWarps = 8;
static_assert(kTsThreads * kTsItems == kSortTile, "sort tile");

// What k_resample_tiles needs of a run (written by k_pair_sort, one coalesced 32-byte load per run).
struct RunInfo {
    uint64_t P;             // joint-CDF prefix of the run's cell (A-25)
    uint64_t bp;            // R_p / n_c of the cell (even split, A-23)
    uint32_t rpm;           // R_p mod n_c
    uint32_t pre;           // rank of the run's first particle among the cell's particles
    uint32_t jbase;         // joint index of the cell's first member (debug)
    uint32_t li;            // the cell's active-list entry
};

struct TilePairs {          // per tile t: entries [t*4096, t*4096 + nd[t])
    uint32_t* key;          // cell key of the run (C = outside the grid)
    uint16_t* first;        // first local sorted position of the run
    uint16_t* cnt;          // particles in the run (1..4096, stored as cnt-1)
    RunInfo* run;           // per-run resampling parameters                           (k_pair_sort)
    uint32_t* nd;           // [tiles] runs of the tile
};

// Stable LSD radix pass over the tile in shared memory: warps own consecutive 512-element slices of
// the current order and rank by 8-bit digit with match_any + running per-warp counters.
__device__ __forceinline__ void tile_radix_pass(uint32_t* s_k, uint16_t* s_i, uint32_t (*s_whist)[256],
                                                uint32_t* s_scan, uint32_t kmin, int shift, uint32_t n)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (int i = tid; i < kTsWarps * 256; i += kTsThreads) (&s_whist[0][0])[i] = 0;
    uint32_t k[kTsItems], rk[kTsItems];
    uint16_t v[kTsItems];
#pragma unroll
    for (int i = 0; i < kTsItems; ++i) {
        const uint32_t p = warp * (kTsItems * 32) + i * 32 + lane;
        k[i] = s_k[p];
        v[i] = s_i[p];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kTsItems; ++i) {
        const uint32_t p = warp * (kTsItems * 32) + i * 32 + lane;
        const bool ok = p < n;
        const uint32_t dig = ok ? (((k[i] - kmin) >> shift) & 255u) : 0x100u;
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
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kTsWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = run;
        run += c;
    }
    uint32_t tot;
    const uint32_t lstart = block_excl_scan<uint32_t, kTsWarps>(run, s_scan, tot);
#pragma unroll
    for (int w = 0; w < kTsWarps; ++w) s_whist[w][tid] += lstart;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kTsItems; ++i) {
        const uint32_t p = warp * (kTsItems * 32) + i * 32 + lane;
        if (p < n) {
            const uint32_t dig = ((k[i] - kmin) >> shift) & 255u;
            const uint32_t pos = s_whist[warp][dig] + rk[i];
            s_k[pos] = k[i];
            s_i[pos] = v[i];
        }
    }
    __syncthreads();
}

__global__ __launch_bounds__(kTsThreads) void k_tilesort(const uint32_t* __restrict__ keys, uint16_t* __restrict__ lperm,
                                                         TilePairs tp, uint32_t* __restrict__ counts,
                                                         uint32_t* __restrict__ npairs, uint32_t nu, uint32_t C)
{
    __shared__ uint32_t s_k[kSortTile];
    __shared__ uint16_t s_i[kSortTile];
    __shared__ uint32_t s_whist[kTsWarps][256];
    __shared__ uint16_t s_start[kSortTile + 1];
    __shared__ uint32_t s_scan[kTsWarps + 1];
    __shared__ uint32_t s_min[kTsWarps], s_max[kTsWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t n = nu > base ? min((uint32_t)kSortTile, nu - base) : 0u;

    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
    for (int i = 0; i < kTsItems / 4; ++i) {
        const uint32_t l = (i * kTsThreads + tid) * 4;
        uint4 k4 = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (l + 3 < n) k4 = *reinterpret_cast<const uint4*>(keys + base + l);
        else {
            if (l < n) k4.x = keys[base + l];
            if (l + 1 < n) k4.y = keys[base + l + 1];
            if (l + 2 < n) k4.z = keys[base + l + 2];
        }
        const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            s_k[l + e] = kk[e];
            s_i[l + e] = (uint16_t)(l + e);
            if (l + e < n) { kmin = min(kmin, kk[e]); kmax = max(kmax, kk[e]); }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, off));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, off));
    }
    if (lane == 0) { s_min[warp] = kmin; s_max[warp] = kmax; }
    __syncthreads();
    kmin = s_min[0]; kmax = s_max[0];
#pragma unroll
    for (int w = 1; w < kTsWarps; ++w) { kmin = min(kmin, s_min[w]); kmax = max(kmax, s_max[w]); }
    const uint32_t range = n ? kmax - kmin : 0u;
    const int bits = range ? 32 - __clz(range) : 0;
    for (int shift = 0; shift < bits; shift += 8) tile_radix_pass(s_k, s_i, s_whist, s_scan, kmin, shift, n);

    // runs of equal keys in sorted order -> pairs
    const uint32_t p0 = tid * kTsItems;
    uint32_t flags = 0, nrun = 0;
#pragma unroll
    for (int i = 0; i < kTsItems; ++i) {
        const uint32_t p = p0 + i;
        const bool head = p < n && (p == 0 || s_k[p] != s_k[p - 1]);
        flags |= (head ? 1u : 0u) << i;
        nrun += head ? 1u : 0u;
    }
    uint32_t nd;
    uint32_t j = block_excl_scan<uint32_t, kTsWarps>(nrun, s_scan, nd);
#pragma unroll
    for (int i = 0; i < kTsItems; ++i)
        if ((flags >> i) & 1u) s_start[j++] = (uint16_t)(p0 + i);
    if (tid == 0) { s_start[nd] = (uint16_t)n; tp.nd[blockIdx.x] = nd; }
    __syncthreads();
    for (uint32_t r = tid; r < nd; r += kTsThreads) {
        const uint32_t f = s_start[r], c = (uint32_t)s_start[r + 1] - f;
        const uint32_t key = s_k[f];
        tp.key[base + r] = key;
        tp.first[base + r] = (uint16_t)f;
        tp.cnt[base + r] = (uint16_t)(c - 1);
        if (key < C) {
            atomicAdd(&counts[key], c);
            atomicAdd(&npairs[key], 1u);
        }
    }
    for (uint32_t p = tid; p < n; p += kTsThreads) lperm[base + p] = s_i[p];
}

// Each pair appends itself (tile << 12 | run) to its cell's list (unordered; k_pair_sort orders it).
__global__ __launch_bounds__(256) void k_pair_fill(TilePairs tp, CellList L, const uint32_t* __restrict__ cell2list,
                                                   uint32_t* __restrict__ plist, uint32_t C)
{
    const uint32_t t = blockIdx.x, base = t * kSortTile;
    const uint32_t nd = tp.nd[t];
    for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x) {
        const uint32_t key = tp.key[base + r];
        if (key >= C) continue;
        const uint32_t li = cell2list[key];
        const uint32_t slot = atomicAdd(&L.pfill[li], 1u);
        plist[L.ps[li] + slot] = (t << 12) | r;
    }
}

// Per active cell: its pair list sorted by tile, then the exclusive prefix of the run counts in that
// order -> pre of every run, and the run's resampling parameters (RunInfo).  Groups of 8 lanes take one
// cell each (4 cells per warp, so neighbouring cells with long lists proceed in parallel); lists are
// staged in shared memory and sorted by rank-by-count (entries are distinct, lists are short).
constexpr int kPsGroup = 8, kPsBuf = 128;

__global__ __launch_bounds__(256) void k_pair_sort(TilePairs tp, CellList L, uint32_t* __restrict__ plist,
                                                   uint32_t* __restrict__ ptmp, const DevScalars* __restrict__ sc)
{
    __shared__ uint32_t s_buf[256 / kPsGroup][2][kPsBuf];
    const int lane = threadIdx.x & 31, gl = lane & (kPsGroup - 1), grp = threadIdx.x / kPsGroup;
    const uint32_t gmask = 0xFFu << (lane & ~(kPsGroup - 1));
    const uint32_t Lc = sc->Lc;
    const uint32_t ng = (gridDim.x * blockDim.x) / kPsGroup;
    for (uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) / kPsGroup; li < Lc; li += ng) {
        const uint32_t m = L.np[li];
        if (m == 0) continue;
        RunInfo ri;
        ri.P = L.P[li];
        ri.bp = L.bp[li];
        ri.rpm = L.rp[li];
        ri.pre = 0u;
        ri.jbase = L.start[li] + L.sb[li];
        ri.li = li;
        uint32_t* pl = plist + L.ps[li];
        if (m == 1) {                                 // (tile << 12 | run) is the run's slot index
            if (gl == 0) tp.run[pl[0]] = ri;
            continue;
        }
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
        // exclusive prefix of counts in tile order
        uint32_t carry = 0;
        for (uint32_t a0 = 0; a0 < mr; a0 += kPsGroup) {
            const uint32_t a = a0 + gl;
            uint32_t v = 0, c = 0;
            if (a < m) {
                v = tmp[a];
                c = (uint32_t)tp.cnt[v] + 1u;
            }
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < kPsGroup; d <<= 1) {
                const uint32_t o = __shfl_up_sync(gmask, incl, d, kPsGroup);
                if (gl >= d) incl += o;
            }
            if (a < m) {
                RunInfo r2 = ri;
                r2.pre = carry + incl - c;
                tp.run[v] = r2;
                pl[a] = v;                   // the cell's list, now in tile order
            }
            carry += __shfl_sync(gmask, incl, kPsGroup - 1, kPsGroup);
        }
        __syncwarp(gmask);
    }
}

}  // namespace dog
