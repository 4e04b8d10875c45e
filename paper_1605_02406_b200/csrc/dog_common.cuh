// dog_common.cuh -- shared device helpers and the per-step device scalar block.
#pragma once
#include <cstdint>

namespace dog {

typedef unsigned __int128 u128;

// Device-resident scalars of the filter (written and read by kernels, so a cycle needs no host sync).
// Every field sits in its own 128-byte line (DS_F): kernels are launched early (PDL) beside their
// predecessor, and an SM's L1 may keep a line a predecessor CTA loaded before another predecessor CTA
// wrote it (griddepcontrol.wait does not invalidate the L1).  No kernel reads a field that another CTA of
// the same kernel writes, so with one field per line no CTA ever caches a line that is written while the
// next kernel can run -- plain L1-cached loads stay coherent without a fence (measured: a gpu-scope fence
// after every wait costs ~7 us per cycle; L2-only loads of the scalars more).
#define DS_F alignas(128)
struct DevScalars {
    DS_F float    w_bar;      // uniform particle weight of the current state S_k (Eq. 57)
    DS_F float    w_pred;     // p_S * w_bar of the cycle in flight (Eq. 39)
    DS_F uint32_t U;          // systematic-resampling offset of the cycle (A-24)
    DS_F uint32_t meas_bad;   // invalid measurement cells seen (sticky until reported)
    DS_F uint64_t W;          // total fixed-point joint weight (A-23)
    DS_F uint64_t A;          // total fixed-point born mass
    DS_F uint64_t n_in;       // particles inside the grid after predict
    DS_F uint64_t s_total;    // birth slots allocated (nu_b or 0)
    DS_F uint32_t n_items;    // birth work items of the cycle
    DS_F uint32_t Lc;         // entries of the active-cell list
    // Local particle array = [migrants from the shard below | own particles | migrants from above]
    // (row-band contexts; a whole-grid context has only own particles).
    DS_F uint32_t n_lo;       // migrants received this cycle from below
    DS_F uint32_t n_hi;       //                          and from above
    DS_F uint32_t n_own[2];   // own particles, indexed by cycle parity
    DS_F uint64_t o_base[2];  // global index of the first own particle (Philox counter base), by parity
    DS_F uint64_t A_acc;      // this context's born mass (k_cells atomics; shared over shards)
    DS_F uint64_t Wtot;       // joint weight over all shards
    DS_F uint64_t Ppre;       // joint prefix of the shards below
    DS_F uint32_t mig_cnt[4]; // migrants leaving this cycle: to the band below, above, further below,
                              // further above (k_pack_migrants; read by the receivers)
    DS_F uint32_t mig_over;   // sticky: a receive exceeded the migrant capacity (cycle not exact)
    DS_F double nu_over_W;    // nu / Wtot in fp64 (k_pair_sort), for the resampling kernels
};

constexpr float kSentinelPos = -1073741824.0f;  // -2^30 cells: empty-world particle (A-19)
constexpr float kMeasSumMax = 0x1.00001p+0f;    // 1 + 2^-20 (= 1.0f + 1e-6f rounded), A-27

// Per-step scalars computed on the host in fp64 and rounded once to f32.
struct StepArgs {
    float Tc;      // T / cell_size: cells moved per (m/s)
    float s_p;     // sigma_pos * T / cell_size: position noise SD in cells (A-1)
    float s_v;     // sigma_vel * T: velocity noise SD in m/s (A-1)
    float alpha;   // exp(-T / free_tau) (A-9)
    int64_t k;     // step counter of the state being advanced
};

struct FilterConst {
    int32_t W, H;
    uint32_t C;          // cells of this context (the band; the whole grid for a whole-grid context)
    uint32_t Cg;         // cells of the whole grid (key of a particle outside the grid)
    uint32_t c_off;      // global index of the context's first cell (row0 * W)
    uint32_t row0;       // first grid row of the context
    uint32_t lo_cap;     // particle slots reserved before the own region (migrants from below)
    uint32_t rank, world;
    uint32_t c_lo, c_hi; // global cells of the neighbour bands [c_lo, c_hi): near / far migrant buckets
    uint32_t nu, nu_b;
    float p_s, p_b, sigma_b, occ_max, v_max;
    uint64_t seed;
    uint32_t force_exact;  // diagnostics (DOG_FORCE_EXACT_F): every F(X) through exact 128-bit products
    double fx, fx_inv;     // 2^FX, 2^-FX: fixed-point scale of the masses (A-23; FX = 40 below 2^24 cells)
};

// Diagnostics build only (DOG_NVCC_EXTRA=-DDOG_TIMING, tools/phase_timing.py): per-phase block time,
// accumulated by thread 0 of every block into g_phase_ns[slot].
#ifdef DOG_TIMING
__device__ unsigned long long g_phase_ns[64];
__device__ __forceinline__ unsigned long long gtimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PHASE_BEGIN() unsigned long long _pt = threadIdx.x == 0 ? gtimer_ns() : 0ull
#define PHASE_MARK(slot) do { if (threadIdx.x == 0) { const unsigned long long _n = gtimer_ns(); \
    atomicAdd(&g_phase_ns[slot], _n - _pt); _pt = _n; } } while (0)
#else
#define PHASE_BEGIN() do { } while (0)
#define PHASE_MARK(slot) do { } while (0)
#endif

// Checked build (DOG_NVCC_EXTRA=-DDOG_CHECKED, tools/checked_tests.sh): device-side bounds assertions on
// the writes whose index comes from a computed prefix (outputs, staging slots, run-list slots).  A
// failed check prints and traps; the release build compiles them out.
#ifdef DOG_CHECKED
#include <cstdio>
#define DOG_ASSERT(cond) do { if (!(cond)) { printf("libdog check failed: %s (%s:%d) block %d thread %d\n", \
    #cond, __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x); __trap(); } } while (0)
#else
#define DOG_ASSERT(cond) do { } while (0)
#endif

// Programmatic dependent launch (every kernel of a cycle is launched with the PDL attribute): a kernel
// lets the next one launch as soon as all its CTAs are running, and waits for its predecessor's results
// (full completion and memory flush) before touching them.  Hides the launch gap between kernels.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// A read of a DevScalars field (see DevScalars: one field per L1 line keeps plain loads coherent).
template <typename T>
__device__ __forceinline__ T scrd(const T& v) { return v; }
#define PDL_ENTER() do { pdl_trigger(); pdl_wait(); } while (0)

// 1-D bulk copy global -> shared (TMA engine, cp.async.bulk), completion counted on an mbarrier as
// transaction bytes; 16-byte aligned addresses, size a multiple of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Calls body(li, m) for every active-list entry with runs (m = np[li] > 0), by groups of G lanes (G a
// power of two <= 32; the group's lanes all call body for the same entry).  kBatch: each group reads G
// consecutive entries per step (one coalesced load) and works through those with runs -- for long lists
// whose entries mostly have none (the exact filter's); otherwise one entry per group per step.
// In batch mode an entry with exactly one run goes to single(li) on its own lane (no group work: the
// exact filter's entries are mostly like that); body(li, m) gets those with two or more.
// kSmall > 1: entries with 1..kSmall runs go to single(li, m) (one lane each), the rest to body.
template <bool kBatch, int G, int kSmall = 1, typename F, typename S1>
__device__ __forceinline__ void for_run_entries(const uint32_t* __restrict__ np, uint32_t Lc, F&& body, S1&& single)
{
    const int lane = threadIdx.x & 31, gl = lane & (G - 1);
    const uint32_t gmask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << (lane & ~(G - 1));
    const uint32_t ng = (gridDim.x * blockDim.x) / G;
    const uint32_t gi = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    if (kBatch) {
        for (uint32_t q0 = gi * G; q0 < Lc; q0 += ng * G) {
            const uint32_t mine = q0 + gl < Lc ? np[q0 + gl] : 0u;
            if constexpr (kSmall == 1) {
                if (mine == 1) single(q0 + gl);
            } else {
                if (mine >= 1 && mine <= (uint32_t)kSmall) single(q0 + gl, mine);
            }
            uint32_t todo = (__ballot_sync(gmask, mine > (uint32_t)kSmall) >> (lane & ~(G - 1))) & (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u));
            while (todo) {
                const int b = __ffs(todo) - 1;
                todo &= todo - 1;
                body(q0 + (uint32_t)b, __shfl_sync(gmask, mine, (lane & ~(G - 1)) + b));
            }
        }
    } else {
        for (uint32_t li = gi; li < Lc; li += ng) {
            const uint32_t m = np[li];
            if (m) body(li, m);
        }
    }
}

// Warp inclusive scan (add) of T via shuffles.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane)
{
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += o;
    }
    return v;
}

// Block exclusive scan for blockDim.x = 32*NW threads; returns exclusive prefix and block total.
template <typename T, int NW>
__device__ __forceinline__ T block_excl_scan(T v, T* s_warp /*[NW]*/, T& total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? s_warp[lane] : T(0);
        T wi = warp_incl_scan(w, lane);
        if (lane < NW) s_warp[lane] = wi - w;   // exclusive warp offsets
        if (lane == NW - 1) s_warp[NW] = wi;    // total
    }
    __syncthreads();
    T res = s_warp[warp] + incl - v;
    total = s_warp[NW];
    __syncthreads();
    return res;
}

}  // namespace dog
