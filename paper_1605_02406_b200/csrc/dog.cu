// dog.cu -- host orchestration and C ABI (include/dog.h) of the B200-native DS-PHD/MIB filter.
//
// One context = one filter on one device.  All state lives in HBM; a cycle is a fixed sequence of
// stream-ordered kernel launches (dog_kernels.cuh) with no host synchronisation: every scalar the
// next stage needs (w_bar, w_pred, W, A, U, n_in) is device-resident (DevScalars).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <new>
#include <utility>
#include <vector>

#include "../../include/dog.h"
#include "dog_kernels.cuh"
#include "dog_sort.cuh"
#include "dog_cells.cuh"
#include "dog_resample.cuh"
#include "dog_ego.cuh"
#include "dog_eval.cuh"
#include "dog_doppler.cuh"

using namespace dog;

namespace {

inline size_t round_up(size_t a, size_t b) { return (a + b - 1) / b * b; }
inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

}  // namespace

struct dog_ctx {
    int device = 0;
    dog_grid grid{};
    dog_params params{};
    uint64_t seed = 0;
    uint32_t flags = 0;
    int64_t nu = 0, nu_b = 0;
    uint32_t C = 0;             // cells of this context (its band)
    uint32_t Cg = 0;            // cells of the whole grid
    int64_t k = 0;
    bool poisoned = false;
    // row band (a whole-grid context is the band [0, H) of a world of one)
    int32_t row0 = 0, row1 = 0, rank = 0, world = 1;
    uint32_t c_lo = 0, c_hi = 0;    // global cells of the neighbour bands
    uint32_t lo_cap = 0, hi_cap = 0, own_cap = 0;   // particle slots: [lo | own | hi]
    size_t nu_cap = 0;          // total particle slots (multiple of the sort tile)
    uint32_t tiles = 0, own_tiles = 0, cell_blocks = 0, cell_chunk = 0, birth_blocks = 0;
    Migrants mg{};              // band contexts: migrants packed for the neighbours
    int phase = 0;              // band cycle: 0 idle, 1 predicted, 2 sizes read, 3 assigned, 4 joint
    float band_dt = 0.0f;

    // state S_k and predicted state (SoA, f32)
    float4* st = nullptr;                         // (x, y, vx, vy) per particle
    float4* pst = nullptr;                        // band contexts: predicted state of the local array (input
                                                  // order, AoS); whole-grid debug builds: the PRED dumps
    float2 *pxy = nullptr, *pv = nullptr;         // predicted state in sorted order, (x, y) and (vx, vy) halves
    // assignment (dog_sort.cuh)
    uint32_t* keys = nullptr;                     // cell key per predicted particle
    uint16_t* lperm = nullptr;                    // tile-local sorted position -> local index
    TilePairs tp{};                               // runs of equal keys per tile
    uint32_t *plist = nullptr, *ptmp = nullptr;   // per-cell run lists
    uint32_t *counts = nullptr, *npairs = nullptr;   // n_c and runs per cell, zeroed by k_cells
    // cells
    float *m_free = nullptr, *occ = nullptr, *fre = nullptr;
    float2* mean = nullptr;
    float* cov = nullptr;
    uint32_t* mvalid = nullptr;                   // moments-reported bitmask
    StageList stage{};                            // k_cells staging (per cell chunk)
    CellList list{};                              // flat active-cell list
    BlockTotals bt{};
    WideScan ws{};                                // grid-wide list scan (large active lists)
    uint32_t ls_cluster = 0, flat_blocks = 0;     // k_list_scan cluster size; lane-per-cell grids
    uint32_t* cell2list = nullptr;
    bool dense = false;                           // this cycle lists every cell at its own index (exact filter)
    MomPartial* ppart = nullptr;                  // velocity sums per run
    // debug-only arrays
    uint32_t* perm = nullptr;
    float *dbg_rho_p = nullptr, *dbg_rho_b = nullptr;
    uint64_t *dbg_Rp = nullptr, *dbg_Rb = nullptr;
    float *bx = nullptr, *by = nullptr, *bvx = nullptr, *bvy = nullptr;
    uint32_t* jidx = nullptr;
    DevScalars* sc = nullptr;
    // end-to-end staging
    float* meas_dev = nullptr;
    // ego-motion compensation (dog_ego_scroll)
    double res_x = 0.0, res_y = 0.0;
    double org_x = 0.0, org_y = 0.0;              // world metres of cell (0, 0)'s lower-left corner
    unsigned long long* ev_counts = nullptr;      // dog_eval_cells results
    EvalAcc* ev_acc = nullptr;                    // dog_eval_cells accumulator (self-resetting)
    double* ev_sums = nullptr;
    float* m_free_tmp = nullptr;
    // pipelined host entry (dog_step_host_async): double-buffered staging, copy streams, events
    float* hmeas[2] = {nullptr, nullptr};
    float* hocc[2] = {nullptr, nullptr};
    cudaStream_t h2d = nullptr, d2h = nullptr;
    // births run on a side stream beside resampling (independent outputs; joined before the step ends)
    // Doppler / association branch (NEXT-1), allocated on the first dog_step_doppler
    uint32_t* kscr = nullptr;                     // k_predict_sort: full keys of tiles with > 2^20-cell boxes
    uint64_t* d_rg = nullptr;                     // per run slot: gfx sum, then exclusive cell prefix
    uint64_t* d_rs = nullptr;                     // per run slot: block prefix at the run's first member
    uint64_t* d_GS = nullptr;                     // per active-list entry: the cell's gfx total (0: none)
    uint8_t* d_tflag = nullptr;                   // per sort tile: holds members of a Doppler cell
    uint32_t* d_gfx = nullptr;                    // per sorted position: g (f32 bits), then fixed-point gfx
    uint32_t* d_gmax = nullptr;                   // per cell: the largest member likelihood (f32 bits, A-34)
    // exact filter with a likelihood (NEXT-3, A-38), allocated on the first dog_step_exact_lik
    uint64_t* d_GSc = nullptr;                    // per cell: sum of the members' gfx (zero between cycles)
    float* d_pAe = nullptr;                       // per cell: effective association weight of the members' split
    float* d_pic = nullptr;                       // per cell: associated share of the births
    const float* band_dop = nullptr;              // band contexts: the cycle's Doppler grid (assign -> resample)
    const float* band_pA = nullptr;
    bool band_exact = false;                      // band contexts: this cycle runs the exact PHD/MIB update
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_used[2] = {}, ev_out[2] = {}, ev_read[2] = {};
    int hbuf = 0;
    // profiling: events[step][stage boundary]
    std::vector<cudaEvent_t> pev;
    int prof_max = 0, prof_steps = 0, prof_nst = 0;
    const char* stage_names[DOG_MAX_STAGES] = {};

    // sharded parent (dog_create with n_devices >= 2): one row-band context per device; the parent holds
    // no particles itself and drives the bands' phases with device-side exchanges (no host sync)
    std::vector<dog_ctx*> shards;
    std::vector<int> shard_dev;
    std::vector<int32_t> shard_rows;              // world + 1 row bounds, bottom-up
    std::vector<cudaStream_t> shard_st;           // internal streams (dog_step on the parent)
    std::vector<cudaEvent_t> sev_pred, sev_asg, sev_jnt, sev_done;
    std::vector<uint64_t*> sh_mass, sh_weight;    // per band, on its device: the all-gathered u64 totals
    cudaEvent_t ev_caller = nullptr;              // on device_ids[0]: the caller's stream -> band streams
    // the active-list length of a recent cycle, copied to pinned host memory at the end of each cycle (no
    // sync; read lagged): long lists (dense scenes, cfg 5) take the grid-wide list scan and the lane-per-cell
    // variants, which produce the same lists / sums as the one-cluster variants
    uint32_t* lc_host = nullptr;

    std::vector<void*> allocs;
};

namespace {

int fail(dog_ctx* c, cudaError_t e, const char* what)
{
    if (c) c->poisoned = true;
    fprintf(stderr, "libdog: %s failed: %s\n", what, cudaGetErrorString(e));
    return DOG_E_CUDA;
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return fail(ctx, _e, #call);   \
    } while (0)
#define CK2(c, call)                                          \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return fail((c), _e, #call);   \
    } while (0)

template <typename T>
int dalloc(dog_ctx* ctx, T** p, size_t n)
{
    void* q = nullptr;
    if (cudaMalloc(&q, n * sizeof(T) > 0 ? n * sizeof(T) : 16) != cudaSuccess) {
        cudaGetLastError();
        return DOG_E_NOMEM;
    }
    ctx->allocs.push_back(q);
    *p = (T*)q;
    return DOG_OK;
}

void free_all(dog_ctx* ctx)
{
    for (void* p : ctx->allocs) cudaFree(p);
    ctx->allocs.clear();
}

bool finite(float v) { return std::isfinite(v); }

// Every kernel of a plain cycle is launched with programmatic stream serialization (PDL, dog_common.cuh):
// its CTAs may start while the previous kernel drains and wait in griddepcontrol.wait for its results.
bool g_pdl = getenv("DOG_NO_PDL") == nullptr;
// Per cycle: run-heavy cycles (the exact filter, dense scenes) launch without PDL -- measured at cfg T:
// their multi-wave kernels ran up to 1.7x slower with the next kernel's CTAs launched early (exact
// cycle 1.39 ms with PDL, 1.21 ms without), while the plain cycle gains ~6 us from it.
thread_local bool t_pdl_cycle = true;
struct PdlScope {
    bool prev;
    explicit PdlScope(bool on) : prev(t_pdl_cycle) { t_pdl_cycle = on; }
    ~PdlScope() { t_pdl_cycle = prev; }
};

template <typename... KArgs, typename... Args>
cudaError_t launch_ex(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      uint32_t cluster, Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    int na = 0;
    if (g_pdl && t_pdl_cycle && pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
    cfg.attrs = at; cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, uint32_t cluster,
                   Args&&... args)
{
    return launch_ex(true, kern, grid, block, smem, st, cluster, std::forward<Args>(args)...);
}

StepArgs step_args(const dog_ctx* ctx, float dt)
{
    // fp64 once, rounded to f32; same expression order as the oracle
    const double T = (double)dt;
    StepArgs a;
    a.Tc = (float)(T / (double)ctx->grid.cell_size);
    a.s_p = (float)(((double)ctx->params.sigma_pos * T) / (double)ctx->grid.cell_size);
    a.s_v = (float)((double)ctx->params.sigma_vel * T);
    a.alpha = (float)std::exp(-(T / (double)ctx->params.free_tau));
    a.k = ctx->k;
    return a;
}

FilterConst filter_const(const dog_ctx* ctx)
{
    FilterConst f;
    f.W = ctx->grid.width;
    f.H = ctx->grid.height;
    f.C = ctx->C;
    f.Cg = ctx->Cg;
    f.c_off = (uint32_t)ctx->row0 * (uint32_t)ctx->grid.width;
    f.row0 = (uint32_t)ctx->row0;
    f.lo_cap = ctx->lo_cap;
    f.rank = (uint32_t)ctx->rank;
    f.world = (uint32_t)ctx->world;
    f.c_lo = ctx->c_lo;
    f.c_hi = ctx->c_hi;
    f.nu = (uint32_t)ctx->nu;
    f.nu_b = (uint32_t)ctx->nu_b;
    f.p_s = ctx->params.p_s;
    f.p_b = ctx->params.p_b;
    f.sigma_b = ctx->params.sigma_birth_vel;
    f.occ_max = ctx->params.occ_max;
    f.v_max = ctx->params.v_max;
    f.seed = ctx->seed;
    f.force_exact = getenv("DOG_FORCE_EXACT_F") ? 1u : 0u;     // diagnostics / tests only
    // fixed-point exponent of the masses (A-23): 40 while the GRID has fewer than 2^24 cells, else 63 minus
    // the bit length of its cell count, so totals over every cell of every band stay below 2^64
    int bits = 0;
    while (bits < 62 && (1ll << bits) <= (int64_t)ctx->grid.width * ctx->grid.height) ++bits;
    const int fxb = bits <= 24 ? 40 : 63 - bits;
    f.fx = std::ldexp(1.0, fxb);
    f.fx_inv = std::ldexp(1.0, -fxb);
    return f;
}

int set_device(dog_ctx* ctx)
{
    if (!ctx->shards.empty()) return DOG_E_STATE;   // a sharded parent: only the dog_*_sharded / state calls
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != ctx->device) CK(cudaSetDevice(ctx->device));
    return DOG_OK;
}

// deferred device-side conditions: a migrant receive beyond capacity (the cycle could not complete
// exactly: the context is poisoned, DOG_E_NOMEM), then invalid measurement cells (DOG_E_MEAS, cleared)
int report_meas(dog_ctx* ctx)
{
    uint32_t bad = 0, over = 0;
    CK(cudaMemcpy(&bad, &ctx->sc->meas_bad, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&over, &ctx->sc->mig_over, 4, cudaMemcpyDeviceToHost));
    if (over) {
        ctx->poisoned = true;
        return DOG_E_NOMEM;
    }
    if (bad) {
        CK(cudaMemset(&ctx->sc->meas_bad, 0, 4));
        return DOG_E_MEAS;
    }
    return DOG_OK;
}

}  // namespace

extern "C" {

int dog_version(void) { return 1; }

const char* dog_error_string(int s)
{
    switch (s) {
    case DOG_OK: return "ok";
    case DOG_E_INVAL: return "invalid argument";
    case DOG_E_NOMEM: return "out of memory";
    case DOG_E_CUDA: return "CUDA error (context poisoned)";
    case DOG_E_NCCL: return "NCCL error (context poisoned)";
    case DOG_E_MEAS: return "invalid measurement cells were treated as vacuous";
    case DOG_E_STATE: return "call-order misuse";
    default: return "unknown status";
    }
}

static int create_impl(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
                       uint64_t seed, uint32_t flags, const dog_band* band, dog_ctx** out)
{
    if (!grid || !params || !out) return DOG_E_INVAL;
    *out = nullptr;
    const dog_params& p = *params;
    const int64_t C = (int64_t)grid->width * grid->height;
    if (grid->width <= 0 || grid->height <= 0 || C >= (1ll << 31) - 1 || !(grid->cell_size > 0.0f) ||
        !finite(grid->cell_size) || grid->width > 65535 || grid->height > 65535)
        return DOG_E_INVAL;   // C < 2^31 - 1 (u32 cell keys, sentinel C); 16-bit rows/cols in the sort keys
    if (n_particles < 1 || n_particles >= (1ll << 30) || n_birth < 0 || n_birth >= (1ll << 30))
        return DOG_E_INVAL;
    if (!(p.p_s > 0.0f && p.p_s <= 1.0f) || !(p.p_b >= 0.0f && p.p_b < 1.0f) ||
        !(p.sigma_pos >= 0.0f) || !finite(p.sigma_pos) || !(p.sigma_vel >= 0.0f) || !finite(p.sigma_vel) ||
        !(p.sigma_birth_vel >= 0.0f) || !finite(p.sigma_birth_vel) || !(p.free_tau > 0.0f) ||
        !(p.occ_max > 0.0f && p.occ_max <= 1.0f) || std::isnan(p.v_max))
        return DOG_E_INVAL;
    if (band && (band->world < 1 || band->rank < 0 || band->rank >= band->world || band->row0 < 0 ||
                 band->row1 <= band->row0 || band->row1 > grid->height || band->lo_row0 > band->row0 ||
                 band->lo_row0 < 0 || band->hi_row1 < band->row1 || band->hi_row1 > grid->height ||
                 (band->rank == 0) != (band->row0 == 0) || (band->rank == band->world - 1) != (band->row1 == grid->height) ||
                 band->migrant_cap == 0 || band->migrant_cap >= (1u << 26)))
        return DOG_E_INVAL;

    dog_ctx* ctx = new (std::nothrow) dog_ctx();
    if (!ctx) return DOG_E_NOMEM;
    cudaGetDevice(&ctx->device);
    ctx->grid = *grid;
    ctx->org_x = (double)grid->origin_x;
    ctx->org_y = (double)grid->origin_y;
    ctx->params = p;
    ctx->seed = seed;
    ctx->flags = flags;
    ctx->nu = n_particles;
    ctx->nu_b = n_birth;
    ctx->Cg = (uint32_t)C;
    if (band && band->world > 1) {
        ctx->row0 = band->row0; ctx->row1 = band->row1; ctx->rank = band->rank; ctx->world = band->world;
        ctx->lo_cap = ctx->hi_cap = (uint32_t)round_up(band->migrant_cap, kSortTile);
        ctx->c_lo = (uint32_t)band->lo_row0 * (uint32_t)grid->width;
        ctx->c_hi = (uint32_t)band->hi_row1 * (uint32_t)grid->width;
    } else {
        ctx->row0 = 0; ctx->row1 = grid->height; ctx->rank = 0; ctx->world = 1;
        ctx->c_lo = 0; ctx->c_hi = (uint32_t)C;
    }
    ctx->C = (uint32_t)(ctx->row1 - ctx->row0) * (uint32_t)grid->width;
    ctx->own_cap = (uint32_t)round_up((size_t)n_particles, kSortTile);
    ctx->nu_cap = (size_t)ctx->lo_cap + ctx->own_cap + ctx->hi_cap;
    ctx->tiles = (uint32_t)(ctx->nu_cap / kSortTile);
    ctx->own_tiles = ctx->own_cap / kSortTile;
    {   // cell chunks of 2048 cells (at most kMaxCellBlocks chunks)
        uint32_t chunk = kCellIter;
        if (const char* e = getenv("DOG_CELL_CHUNK"))       // diagnostics: a multiple of 2048 cells
            chunk = std::max<uint32_t>(kCellIter, (uint32_t)atoi(e) / kCellIter * kCellIter);
        uint32_t nblk = cdiv(ctx->C, chunk);
        while (nblk > (uint32_t)kMaxCellBlocks) { chunk *= 2; nblk = cdiv(ctx->C, chunk); }
        ctx->cell_chunk = chunk;
        ctx->cell_blocks = nblk;
    }
    cudaFuncSetAttribute(k_predict_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPsSmemBytes);
    cudaFuncSetAttribute(k_predict_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPsSmemBytes);
    cudaFuncSetAttribute(k_resample_tiles<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRtSmemBytes);
    cudaFuncSetAttribute(k_resample_tiles<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRtSmemBytes);
    cudaFuncSetAttribute(k_eval_cells_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEvSmem);
    cudaFuncSetAttribute(k_resample_dopp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRdSmemBytes);
    if (const char* cv = getenv("DOG_RS_CARVEOUT")) {   // experiments: shared-memory share of the L1/smem array
        cudaFuncSetAttribute(k_resample_tiles<false>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        cudaFuncSetAttribute(k_resample_tiles<true>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
    }
    {   // persistent grids: as many blocks as fit on the GPU at once
        int per_sm = 0, sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_births, 256, 0);
        ctx->birth_blocks = (uint32_t)std::max(1, per_sm) * (uint32_t)sms;
        ctx->flat_blocks = 4u * (uint32_t)sms;   // lane-per-cell kernels over the active list
        // k_list_scan: one cluster, 16 CTAs where the GPU allows it (non-portable size), else 8
        cudaFuncSetAttribute(k_list_scan, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (uint32_t ncl : {(uint32_t)kLsClusterMax, 8u}) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = ncl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(ncl); cfg.blockDim = dim3(kLsThreads); cfg.attrs = at; cfg.numAttrs = 1;
            int ncls = 0;
            if (cudaOccupancyMaxActiveClusters(&ncls, k_list_scan, &cfg) == cudaSuccess && ncls > 0) {
                ctx->ls_cluster = ncl;
                break;
            }
            cudaGetLastError();
        }
        if (!ctx->ls_cluster) {
            fprintf(stderr, "libdog: no thread-block cluster configuration fits k_list_scan\n");
            delete ctx;
            return DOG_E_CUDA;
        }
    }
    const size_t N = ctx->nu_cap, NB = (size_t)(n_birth > 0 ? n_birth : 1), Cs = (size_t)ctx->C;
    const bool dbg = (flags & DOG_FLAG_DEBUG) != 0;

    int rc = DOG_OK;
#define AL(ptr, n) \
    if (rc == DOG_OK) rc = dalloc(ctx, &ptr, (n))
    AL(ctx->st, N); AL(ctx->pxy, N); AL(ctx->pv, N);
    if (dbg || (band && band->world > 1)) AL(ctx->pst, N);
    AL(ctx->lperm, N); AL(ctx->kscr, N);
    AL(ctx->tp.key, N); AL(ctx->tp.first, N); AL(ctx->tp.cnt, N); AL(ctx->tp.run, N); AL(ctx->tp.nd, ctx->tiles);
    AL(ctx->plist, N); AL(ctx->ptmp, N); AL(ctx->ppart, N);
    AL(ctx->counts, Cs + 1); AL(ctx->npairs, Cs + 1);
    if (dbg) {
        AL(ctx->keys, N); AL(ctx->perm, N); AL(ctx->jidx, N);
        AL(ctx->dbg_rho_p, Cs); AL(ctx->dbg_rho_b, Cs); AL(ctx->dbg_Rp, Cs); AL(ctx->dbg_Rb, Cs);
        AL(ctx->bx, NB); AL(ctx->by, NB); AL(ctx->bvx, NB); AL(ctx->bvy, NB);
    }
    AL(ctx->m_free, Cs); AL(ctx->occ, Cs); AL(ctx->fre, Cs);
    if (ctx->world == 1) AL(ctx->m_free_tmp, Cs);   // ego-motion compensation scrolls into it
    AL(ctx->ev_counts, 4 * kEvalMaxThr); AL(ctx->ev_sums, 5); AL(ctx->ev_acc, 1);
    AL(ctx->mean, Cs); AL(ctx->cov, 3 * Cs);
    AL(ctx->mvalid, Cs / 32 + 1);
    const size_t LC = (size_t)ctx->cell_blocks * ctx->cell_chunk;   // staging capacity >= C
    AL(ctx->stage.c, LC); AL(ctx->stage.n, LC); AL(ctx->stage.Rp, LC); AL(ctx->stage.Rb, LC);
    AL(ctx->stage.rho_p, LC); AL(ctx->stage.np, LC);
    AL(ctx->list.c, Cs); AL(ctx->list.n, Cs); AL(ctx->list.Rp, Cs); AL(ctx->list.rho_p, Cs);
    AL(ctx->list.start, Cs); AL(ctx->list.sb, Cs); AL(ctx->list.nb, Cs); AL(ctx->list.P, Cs); AL(ctx->list.brec, Cs);
    AL(ctx->list.it, Cs); AL(ctx->list.bp, Cs); AL(ctx->list.rp, Cs); AL(ctx->list.bb, Cs);
    AL(ctx->list.rb, Cs); AL(ctx->list.np, Cs); AL(ctx->list.ps, Cs); AL(ctx->list.pfill, Cs);
    AL(ctx->cell2list, Cs);
    AL(ctx->bt.cnt, ctx->cell_blocks); AL(ctx->bt.n0, ctx->cell_blocks); AL(ctx->bt.rb0, ctx->cell_blocks);
    AL(ctx->bt.np0, ctx->cell_blocks);
    AL(ctx->ws.pcnt, ctx->cell_blocks); AL(ctx->ws.pn, ctx->cell_blocks); AL(ctx->ws.pnp, ctx->cell_blocks);
    AL(ctx->ws.prb, ctx->cell_blocks); AL(ctx->ws.tJ, ctx->cell_blocks); AL(ctx->ws.tit, ctx->cell_blocks);
    AL(ctx->ws.pJ, ctx->cell_blocks); AL(ctx->ws.pit, ctx->cell_blocks);

    if (ctx->world > 1) {
        for (int d = 0; d < kMigDirs; ++d) {
            AL(ctx->mg.scr[d], ctx->own_cap); AL(ctx->mg.cnt[d], ctx->own_tiles); AL(ctx->mg.send[d], ctx->lo_cap);
        }
        ctx->mg.cap = ctx->lo_cap;
    }
    AL(ctx->sc, 1);
#undef AL
    if (rc != DOG_OK) {
        free_all(ctx);
        delete ctx;
        return rc;
    }

    // empty initial state (A-19): sentinel particles of weight 0, m_F = 0, k = 0 (a band context starts
    // with no own particles: the sentinels contribute nothing to any band)
    std::vector<float4> sent(N, make_float4(kSentinelPos, kSentinelPos, 0.0f, 0.0f));
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMemcpy(ctx->st, sent.data(), N * 16, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(ctx->m_free, 0, Cs * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->occ, 0, Cs * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->fre, 0, Cs * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->mean, 0, Cs * 8);
    if (e == cudaSuccess) e = cudaMemset(ctx->cov, 0, Cs * 12);
    if (e == cudaSuccess) e = cudaMemset(ctx->sc, 0, sizeof(DevScalars));
    if (e == cudaSuccess) {
        const uint32_t own0[2] = {ctx->world > 1 ? 0u : (uint32_t)n_particles, ctx->world > 1 ? 0u : (uint32_t)n_particles};
        e = cudaMemcpy(ctx->sc->n_own, own0, sizeof(own0), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMemset(ctx->counts, 0, (Cs + 1) * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->npairs, 0, (Cs + 1) * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->mvalid, 0, (Cs / 32 + 1) * 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->ev_acc, 0, sizeof(EvalAcc));

    if (e == cudaSuccess && ctx->world == 1 && ctx->nu_b > 0 && !getenv("DOG_NO_FORK")) {
        if (cudaHostAlloc((void**)&ctx->lc_host, 16, cudaHostAllocDefault) == cudaSuccess) *ctx->lc_host = 0u;
        else { ctx->lc_host = nullptr; cudaGetLastError(); }
        e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "libdog: dog_create init failed: %s\n", cudaGetErrorString(e));
        free_all(ctx);
        delete ctx;
        return DOG_E_CUDA;
    }
    *out = ctx;
    return DOG_OK;
}

static int create_sharded(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
                          uint64_t seed, uint32_t flags, int n_devices, const int* device_ids, dog_ctx** out);

int dog_create(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
               uint64_t seed, uint32_t flags, int n_devices, const int* device_ids, dog_ctx** out)
{
    if (!out || n_devices < 0 || (n_devices > 0 && !device_ids)) return DOG_E_INVAL;
    if (n_devices >= 2)
        return create_sharded(grid, n_particles, n_birth, params, seed, flags, n_devices, device_ids, out);
    int prev = -1;
    cudaGetDevice(&prev);
    if (n_devices == 1 && cudaSetDevice(device_ids[0]) != cudaSuccess) {
        cudaGetLastError();
        return DOG_E_INVAL;
    }
    const int rc = create_impl(grid, n_particles, n_birth, params, seed, flags, nullptr, out);
    if (prev >= 0) cudaSetDevice(prev);
    return rc;
}

int dog_create_band(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
                    uint64_t seed, uint32_t flags, const dog_band* band, dog_ctx** out)
{
    if (!band) return DOG_E_INVAL;
    if (flags & DOG_FLAG_DEBUG) return DOG_E_INVAL;   // stage dumps are whole-grid only
    return create_impl(grid, n_particles, n_birth, params, seed, flags, band, out);
}

static void free_doppler(dog_ctx* ctx);

static int destroy_sharded(dog_ctx* ctx);

int dog_destroy(dog_ctx* ctx)
{
    if (!ctx) return DOG_E_INVAL;
    if (!ctx->shards.empty()) return destroy_sharded(ctx);
    set_device(ctx);
    cudaDeviceSynchronize();
    for (cudaEvent_t e : ctx->pev) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t e : {ctx->ev_in[b], ctx->ev_used[b], ctx->ev_out[b], ctx->ev_read[b]})
            if (e) cudaEventDestroy(e);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->lc_host) cudaFreeHost(ctx->lc_host);
    free_doppler(ctx);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    free_all(ctx);
    delete ctx;
    return DOG_OK;
}

int dog_launches_per_step(dog_ctx* ctx)
{
    if (!ctx) return DOG_E_INVAL;
    if (!ctx->shards.empty()) return DOG_E_STATE;
    // predict_sort, cells, list_scan, pair_fill, pair_sort, resample_tiles, moments, births
    return ctx->nu_b > 0 ? 8 : 7;
}

// ---- the kernels of one cycle (shared by the whole-grid step and the band phases)
static int L_predict_sort(dog_ctx* ctx, bool fused, const StepArgs& a, const FilterConst& fc, cudaStream_t st)
{
    const bool dbg = (ctx->flags & DOG_FLAG_DEBUG) != 0;
    if (fused)
        CK(launch(k_predict_sort<true>, ctx->tiles, kPsThreads, kPsSmemBytes, st, 0, (const float4*)ctx->st,
                  dbg ? ctx->pst : nullptr, ctx->pxy, ctx->pv, dbg ? ctx->keys : nullptr, dbg ? ctx->lperm : nullptr,
                  ctx->tp, ctx->counts, ctx->npairs, ctx->sc, fc, a, ctx->kscr));
    else
        CK(launch(k_predict_sort<false>, ctx->tiles, kPsThreads, kPsSmemBytes, st, 0, (const float4*)ctx->st, ctx->pst,
                  ctx->pxy, ctx->pv, (uint32_t*)nullptr, (uint16_t*)nullptr, ctx->tp, ctx->counts, ctx->npairs, ctx->sc,
                  fc, a, ctx->kscr));
    return DOG_OK;
}

static int L_cells(dog_ctx* ctx, const float* meas, const StepArgs& a, const FilterConst& fc, cudaStream_t st,
                   const float* obs = nullptr, const ExactLik& xl = ExactLik{})
{
    const bool dbg = (ctx->flags & DOG_FLAG_DEBUG) != 0;
    CellDebug cdbg{dbg ? ctx->dbg_rho_p : nullptr, ctx->dbg_rho_b, ctx->dbg_Rp, ctx->dbg_Rb};
    // dense cycles stage every cell at its own index directly into the list arrays (~all cells are active
    // in the exact filter: no compaction, no copy to the list, cell -> entry is the identity)
    const StageList sl = ctx->dense ? StageList{ctx->list.c, ctx->list.n, ctx->list.Rp, ctx->stage.Rb, ctx->list.rho_p,
                                                ctx->list.np}
                                    : ctx->stage;
    if (obs)
        CK(launch(k_cells<true>, ctx->cell_blocks, kCellThreads, 0, st, 0, ctx->counts, ctx->npairs, ctx->m_free,
                  (const float2*)nullptr, ctx->occ, ctx->fre, ctx->mean, ctx->cov, ctx->mvalid, cdbg, sl, ctx->bt,
                  ctx->cell_chunk, ctx->sc, fc, a.alpha, (const float4*)obs, xl, (uint32_t)ctx->dense));
    else
        CK(launch(k_cells<false>, ctx->cell_blocks, kCellThreads, 0, st, 0, ctx->counts, ctx->npairs, ctx->m_free,
                  (const float2*)meas, ctx->occ, ctx->fre, ctx->mean, ctx->cov, ctx->mvalid, cdbg, sl, ctx->bt,
                  ctx->cell_chunk, ctx->sc, fc, a.alpha, (const float4*)nullptr, xl, (uint32_t)ctx->dense));
    return DOG_OK;
}

static int L_list_scan(dog_ctx* ctx, const uint64_t* A_all, const StepArgs& a, const FilterConst& fc, cudaStream_t st,
                       bool wide = false)
{
    if (wide) {   // every cell may be active (exact filter): grid-wide scan over k_cells' chunks
        CK(launch(k_ls_prefix1, 1, 1024, 0, st, 0, ctx->bt, ctx->cell_blocks, ctx->ws, ctx->sc, A_all, fc));
        const StageList sl = ctx->dense ? StageList{ctx->list.c, ctx->list.n, ctx->list.Rp, ctx->stage.Rb, ctx->list.rho_p,
                                                    ctx->list.np}
                                        : ctx->stage;
        CK(launch(k_ls_chunks1, ctx->cell_blocks, 256, 0, st, 0, sl, ctx->list, ctx->bt, ctx->cell_chunk,
                  ctx->cell2list, ctx->ws, (const DevScalars*)ctx->sc, fc, (uint32_t)ctx->dense));
        CK(launch(k_ls_prefix2, 1, 1024, 0, st, 0, ctx->cell_blocks, ctx->ws));
        CK(launch(k_ls_chunks2, ctx->cell_blocks, 256, 0, st, 0, ctx->list, ctx->bt, ctx->ws, ctx->sc, fc,
                  (int64_t)a.k));
        return DOG_OK;
    }
    CK(launch(k_list_scan, ctx->ls_cluster, kLsThreads, 0, st, ctx->ls_cluster, ctx->stage, ctx->list, ctx->bt,
              ctx->cell_blocks, ctx->cell_chunk, ctx->cell2list, A_all, ctx->sc, fc, (int64_t)a.k));
    return DOG_OK;
}

static int L_pairs(dog_ctx* ctx, const uint64_t* W_all, const StepArgs& a, const FilterConst& fc, cudaStream_t st,
                   bool long_list = false, DopPS dp = DopPS{nullptr, nullptr, nullptr, nullptr, nullptr})
{
    CK(launch(k_pair_fill, ctx->tiles, 256, 0, st, 0, ctx->tp, ctx->list,
              ctx->dense ? (const uint32_t*)nullptr : (const uint32_t*)ctx->cell2list, ctx->plist, ctx->C));
    if (long_list)   // every cell listed, most without runs (the exact filter)
        CK(launch(k_pair_sort<true>, 2 * ctx->flat_blocks, 256, 0, st, 0, ctx->tp, ctx->list, ctx->plist, ctx->ptmp, W_all,
                  ctx->sc, fc, (int)(a.k & 1), dp));
    else
        CK(launch(k_pair_sort<false>, ctx->flat_blocks, 256, 0, st, 0, ctx->tp, ctx->list, ctx->plist, ctx->ptmp, W_all,
                  ctx->sc, fc, (int)(a.k & 1), dp));
    return DOG_OK;
}

static int L_resample(dog_ctx* ctx, const StepArgs& a, const FilterConst& fc, cudaStream_t st,
                      const uint64_t* dopGS = nullptr, bool long_list = false)
{
    const bool dbg = (ctx->flags & DOG_FLAG_DEBUG) != 0;
    NextState ns{ctx->st, dbg ? ctx->jidx : nullptr};
    const int par = (int)(a.k & 1);
    static const bool rs_pdl = getenv("DOG_RS_NOPDL") == nullptr;   // diagnostics
    if (dbg)
        CK(launch_ex(rs_pdl, k_resample_tiles<true>, ctx->tiles, kRtThreads, kRtSmemBytes, st, 0, (const uint16_t*)ctx->lperm,
                  ctx->tp, (const float2*)ctx->pxy, (const float2*)ctx->pv, ctx->list, ns, ctx->perm, ctx->ppart,
                  (const DevScalars*)ctx->sc, fc, par, dopGS, long_list ? kMoDirect : 0u));
    else
        CK(launch_ex(rs_pdl, k_resample_tiles<false>, ctx->tiles, kRtThreads, kRtSmemBytes, st, 0, (const uint16_t*)nullptr,
                  ctx->tp, (const float2*)ctx->pxy, (const float2*)ctx->pv, ctx->list, ns, (uint32_t*)nullptr, ctx->ppart,
                  (const DevScalars*)ctx->sc, fc, par, dopGS, long_list ? kMoDirect : 0u));
    return DOG_OK;
}

static int L_moments(dog_ctx* ctx, cudaStream_t st, const uint64_t* GSd = nullptr, bool long_list = false)
{
    const FilterConst fc = filter_const(ctx);
    if (long_list)
        CK(launch(k_moments<true>, 2 * ctx->flat_blocks, 256, 0, st, 0, ctx->list, ctx->tp, (const uint32_t*)ctx->plist,
                  (const float2*)ctx->pv, (const MomPartial*)ctx->ppart, ctx->mean, ctx->cov, (const DevScalars*)ctx->sc,
                  fc, GSd));
    else
        CK(launch(k_moments<false>, ctx->flat_blocks, 256, 0, st, 0, ctx->list, ctx->tp, (const uint32_t*)ctx->plist,
                  (const float2*)ctx->pv, (const MomPartial*)ctx->ppart, ctx->mean, ctx->cov, (const DevScalars*)ctx->sc,
                  fc, GSd));
    return DOG_OK;
}

static int L_births(dog_ctx* ctx, const StepArgs& a, const FilterConst& fc, cudaStream_t st,
                    const DopIn* din = nullptr, bool per_slot = false, const BirthLik& bl = BirthLik{})
{
    if (ctx->nu_b == 0) return DOG_OK;
    const bool dbg = (ctx->flags & DOG_FLAG_DEBUG) != 0;
    NextState ns{ctx->st, dbg ? ctx->jidx : nullptr};
    BirthDebug bd{dbg ? ctx->bx : nullptr, ctx->by, ctx->bvx, ctx->bvy};
    if (per_slot)
        CK(launch(k_births_slots, (uint32_t)std::max<int64_t>(1, std::min<int64_t>((ctx->nu_b + 255) / 256, 8 * 148)), 256, 0,
                  st, 0, ctx->list, ns, bd, (const DevScalars*)ctx->sc, fc, (int64_t)a.k, bl));
    else
        CK(launch(k_births, ctx->birth_blocks, 256, 0, st, 0, ctx->list, ns, bd, (const DevScalars*)ctx->sc, fc,
                  (int64_t)a.k, din ? din->pA : (const float*)nullptr, din ? din->dop : (const float4*)nullptr));
    return DOG_OK;
}

static int step_impl(dog_ctx* ctx, const float* meas, const float* obs, float dt, void* stream);

static int step_parent(dog_ctx* ctx, const float* meas, float dt, void* stream);

int dog_step(dog_ctx* ctx, const float* meas, float dt, void* stream)
{
    if (!meas) return DOG_E_INVAL;
    if (ctx && !ctx->shards.empty()) return step_parent(ctx, meas, dt, stream);
    return step_impl(ctx, meas, nullptr, dt, stream);
}

int dog_step_exact(dog_ctx* ctx, const float* obs, float dt, void* stream)
{
    if (!obs || ((uintptr_t)obs & 15u) != 0) return DOG_E_INVAL;
    return step_impl(ctx, nullptr, obs, dt, stream);
}

static int step_impl(dog_ctx* ctx, const float* meas, const float* obs, float dt, void* stream)
{
    if (!ctx) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1) return DOG_E_STATE;                 // band contexts run the dog_band_* phases
    if (!(dt > 0.0f) || !finite(dt)) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const StepArgs a = step_args(ctx, dt);
    const FilterConst fc = filter_const(ctx);

    // run-heavy cycle: the exact filter, or a dense scene by the lagged list length
    static const uint32_t heavy_div = getenv("DOG_HEAVY_DIV") ? (uint32_t)atoi(getenv("DOG_HEAVY_DIV")) : 4u;
    const bool heavy = obs != nullptr || (ctx->lc_host && *(volatile uint32_t*)ctx->lc_host > ctx->C / heavy_div);
    static const bool heavy_pdl = getenv("DOG_HEAVY_PDL") != nullptr;   // diagnostics
    const PdlScope pdl_scope(!heavy || heavy_pdl);
    ctx->dense = obs != nullptr;                            // the exact filter: every cell is active
    const bool prof = ctx->prof_steps < ctx->prof_max;
    int mark_i = 0;
    auto mark = [&](const char* name) -> cudaError_t {
        if (!prof) return cudaSuccess;
        if (mark_i > 0) ctx->stage_names[mark_i - 1] = name;
        return cudaEventRecord(ctx->pev[(size_t)ctx->prof_steps * (DOG_MAX_STAGES + 1) + mark_i++], st);
    };
    CK(mark(nullptr));
    // 1-2. predict (Alg. 1) fused with the tile-local stable sort (Alg. 2): runs, per-cell counts
    if (int r = L_predict_sort(ctx, true, a, fc, st)) return r;
    CK(mark("predict_sort"));
    // 3. cells: DS predict/update, birth split, fixed point, active-cell staging (Alg. 3)
    if (int r = L_cells(ctx, meas, a, fc, st, obs)) return r;
    CK(mark("cells"));
    // 4. flat active list: slots, joint CDF, run-list offsets (Alg. 5 / Alg. 7 prefix sums), one cluster
    static const int hv = getenv("DOG_HEAVY") ? atoi(getenv("DOG_HEAVY")) : 15;   // diagnostics: which parts
    const bool h_scan = obs != nullptr || (heavy && (hv & 1)), h_pairs = obs != nullptr || (heavy && (hv & 2));
    const bool h_mom = obs != nullptr || (heavy && (hv & 4)), h_births = obs != nullptr || (heavy && (hv & 8));
    if (int r = L_list_scan(ctx, nullptr, a, fc, st, h_scan)) return r;
    CK(mark("list_scan"));
    // 5. each cell's runs in tile order -> stable within-cell ranks; global totals (w_bar)
    if (int r = L_pairs(ctx, nullptr, a, fc, st, h_pairs)) return r;
    CK(mark("pairs"));
    // 6. persistent particles: moments + resampling copies; births.  Births depend only on the list and
    // the totals (both final here) and write disjoint output slots, so outside profiling they run on the
    // side stream concurrently with resampling and are joined before the step ends.
    const bool fork = ctx->side && !prof;
    if (fork) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        if (ctx->lc_host) CK(cudaMemcpyAsync(ctx->lc_host, &ctx->sc->Lc, 4, cudaMemcpyDeviceToHost, ctx->side));
        if (int r = L_births(ctx, a, fc, ctx->side, nullptr, h_births)) return r;
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
    }
    if (int r = L_resample(ctx, a, fc, st, nullptr, h_mom)) return r;
    CK(mark("resample"));
    if (int r = L_moments(ctx, st, nullptr, h_mom)) return r;
    CK(mark("moments"));
    if (fork) {
        CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    } else {
        if (int r = L_births(ctx, a, fc, st, nullptr, h_births)) return r;
        CK(mark("births"));
    }
    if (prof) {
        ctx->prof_nst = mark_i - 1;
        ctx->prof_steps += 1;
    }
    ctx->k += 1;
    return DOG_OK;
}

// Doppler working buffers, allocated on first use; a partial failure frees them all (the next call retries)
static void free_doppler(dog_ctx* ctx)
{
    for (void** p : {(void**)&ctx->d_rg, (void**)&ctx->d_rs, (void**)&ctx->d_GS, (void**)&ctx->d_tflag,
                     (void**)&ctx->d_gfx, (void**)&ctx->d_gmax, (void**)&ctx->d_GSc, (void**)&ctx->d_pAe,
                     (void**)&ctx->d_pic}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
}

static int alloc_doppler(dog_ctx* ctx)
{
    if (ctx->d_rg && ctx->d_rs && ctx->d_GS && ctx->d_tflag && ctx->d_gfx && ctx->d_gmax) return DOG_OK;
    free_doppler(ctx);
    if (cudaMalloc(&ctx->d_rg, ctx->nu_cap * 8) != cudaSuccess || cudaMalloc(&ctx->d_rs, ctx->nu_cap * 8) != cudaSuccess ||
        cudaMalloc(&ctx->d_GS, (size_t)ctx->C * 8) != cudaSuccess || cudaMalloc(&ctx->d_tflag, ctx->tiles) != cudaSuccess ||
        cudaMalloc(&ctx->d_gfx, ctx->nu_cap * 4) != cudaSuccess || cudaMalloc(&ctx->d_gmax, (size_t)ctx->C * 4) != cudaSuccess ||
        cudaMemset(ctx->d_gmax, 0, (size_t)ctx->C * 4) != cudaSuccess) {
        free_doppler(ctx);
        cudaGetLastError();
        return DOG_E_NOMEM;
    }
    return DOG_OK;
}

// the members' likelihoods g, the cell maxima g_max, then gfx relative to g_max summed per run (A-34)
static int L_dopp_runs(dog_ctx* ctx, const DopIn& din, const FilterConst& fc, int par, cudaStream_t st,
                       uint64_t* gsc = nullptr)
{
    // (d_gmax is zero here: zeroed at allocation, and k_pair_sort clears every cell it set)
    CK(launch(k_dopp_g, ctx->tiles, 256, 0, st, 0, ctx->tp, (const float2*)ctx->pv, din,
              ctx->d_gmax, ctx->d_gfx, (const DevScalars*)ctx->sc, fc, par));
    CK(launch(k_dopp_runs, ctx->tiles, 256, 0, st, 0, ctx->tp, din, (const uint32_t*)ctx->d_gmax, ctx->d_rg,
              ctx->d_tflag, ctx->d_gfx, (const DevScalars*)ctx->sc, fc, par, gsc));
    return DOG_OK;
}

// ---- Doppler / association branch (NEXT-1): the cycle with per-member weights in Doppler cells
int dog_step_doppler(dog_ctx* ctx, const float* meas, const float* doppler, const float* p_assoc, float dt,
                     void* stream)
{
    if (!ctx || !meas || !doppler || !p_assoc) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1) return DOG_E_STATE;                 // whole-grid contexts only
    if (!(dt > 0.0f) || !finite(dt)) return DOG_E_INVAL;
    if (((uintptr_t)doppler & 15u) != 0) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    if (int r = alloc_doppler(ctx)) return r;
    const StepArgs a = step_args(ctx, dt);
    const FilterConst fc = filter_const(ctx);
    const DopIn din{(const float4*)doppler, p_assoc};
    const int par = (int)(a.k & 1);
    ctx->dense = false;
    if (int r = L_predict_sort(ctx, true, a, fc, st)) return r;
    // the per-run likelihood sums need only the tile sort: on the side stream beside k_cells and the
    // list scan (they touch nothing it reads or writes), joined before the pair sort consumes them
    const bool fork = ctx->side != nullptr;
    cudaStream_t ds = fork ? ctx->side : st;
    if (fork) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    }
    if (int r = L_dopp_runs(ctx, din, fc, par, ds)) return r;
    if (fork) CK(cudaEventRecord(ctx->ev_join, ctx->side));
    if (int r = L_cells(ctx, meas, a, fc, st)) return r;
    if (int r = L_list_scan(ctx, nullptr, a, fc, st)) return r;
    if (fork) CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    // the pair sort also turns the run sums into in-cell prefixes, the cell totals GS and the tile flags
    if (int r = L_pairs(ctx, nullptr, a, fc, st, false, DopPS{p_assoc, ctx->d_rg, ctx->d_GS, ctx->d_tflag, ctx->d_gmax})) return r;
    if (fork) {   // births beside the resampling (disjoint output slots), as in dog_step
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        if (int r = L_births(ctx, a, fc, ctx->side, &din)) return r;
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
    }
    // tiles without a Doppler cell's members: the closed-form kernel; the others: per-member weights
    if (int r = L_resample(ctx, a, fc, st, ctx->d_GS)) return r;
    NextState ns{ctx->st, nullptr};
    CK(launch_ex(false, k_resample_dopp, ctx->tiles, 256, kRdSmemBytes, st, 0, ctx->tp,
                 (const float2*)ctx->pxy, (const float2*)ctx->pv, ctx->list, ns, ctx->ppart, din, (const uint64_t*)ctx->d_rg, ctx->d_rs,
                 (const uint64_t*)ctx->d_GS, (const uint8_t*)ctx->d_tflag, (const uint32_t*)ctx->d_gfx,
                 (const DevScalars*)ctx->sc, fc, par));
    if (int r = L_moments(ctx, st, ctx->d_GS)) return r;
    if (fork) CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    else if (int r = L_births(ctx, a, fc, st, &din)) return r;
    ctx->k += 1;
    return DOG_OK;
}

// ---- exact filter with a single-object likelihood (NEXT-3 general form, A-38): the members'
// likelihoods and their per-cell sums come first (the cell update needs them), then the exact cycle
// with the Doppler split in the likelihood cells.
static int alloc_lik(dog_ctx* ctx)
{
    if (int r = alloc_doppler(ctx)) return r;
    if (ctx->d_GSc && ctx->d_pAe && ctx->d_pic) return DOG_OK;
    for (void** p : {(void**)&ctx->d_GSc, (void**)&ctx->d_pAe, (void**)&ctx->d_pic}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    if (cudaMalloc(&ctx->d_GSc, (size_t)ctx->C * 8) != cudaSuccess || cudaMalloc(&ctx->d_pAe, (size_t)ctx->C * 4) != cudaSuccess ||
        cudaMalloc(&ctx->d_pic, (size_t)ctx->C * 4) != cudaSuccess ||
        cudaMemset(ctx->d_GSc, 0, (size_t)ctx->C * 8) != cudaSuccess) {   // k_cells clears what it reads
        free_doppler(ctx);
        cudaGetLastError();
        return DOG_E_NOMEM;
    }
    return DOG_OK;
}

int dog_step_exact_lik(dog_ctx* ctx, const float* obs, const float* lik, const float* p_assoc, float dt, void* stream)
{
    if (!ctx || !obs || !lik || !p_assoc) return DOG_E_INVAL;
    if (((uintptr_t)obs & 15u) != 0 || ((uintptr_t)lik & 15u) != 0) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1) return DOG_E_STATE;                 // whole-grid contexts only
    if (!(dt > 0.0f) || !finite(dt)) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    if (int r = alloc_lik(ctx)) return r;
    const StepArgs a = step_args(ctx, dt);
    const FilterConst fc = filter_const(ctx);
    const int par = (int)(a.k & 1);
    const PdlScope pdl_scope(false);                        // a run-heavy cycle (see t_pdl_cycle)
    ctx->dense = true;                                      // every cell listed at its own index
    // gated: only cells where a measurement occurred carry the likelihood
    const DopIn dg{(const float4*)lik, p_assoc, (const float4*)obs};
    if (int r = L_predict_sort(ctx, true, a, fc, st)) return r;
    if (int r = L_dopp_runs(ctx, dg, fc, par, st, ctx->d_GSc)) return r;
    const ExactLik xl{p_assoc, (const float4*)lik, ctx->d_GSc, (const uint32_t*)ctx->d_gmax, ctx->d_pAe, ctx->d_pic};
    if (int r = L_cells(ctx, nullptr, a, fc, st, obs, xl)) return r;
    if (int r = L_list_scan(ctx, nullptr, a, fc, st, true)) return r;
    // run sums are nonzero only in the gated cells, so the ungated p_A marks the same Doppler cells
    if (int r = L_pairs(ctx, nullptr, a, fc, st, true, DopPS{p_assoc, ctx->d_rg, ctx->d_GS, ctx->d_tflag, ctx->d_gmax})) return r;
    const BirthLik bl{p_assoc, (const float4*)obs, (const float4*)lik, ctx->d_pic};
    const bool fork = ctx->side != nullptr;
    if (fork) {   // births beside the resampling (disjoint output slots), as in dog_step
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        if (int r = L_births(ctx, a, fc, ctx->side, nullptr, true, bl)) return r;
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
    }
    if (int r = L_resample(ctx, a, fc, st, ctx->d_GS, true)) return r;
    // the members' split weight in the likelihood cells is the effective pAe (A-38)
    const DopIn de{(const float4*)lik, ctx->d_pAe, nullptr};
    NextState ns{ctx->st, nullptr};
    CK(launch_ex(false, k_resample_dopp, ctx->tiles, 256, kRdSmemBytes, st, 0, ctx->tp,
                 (const float2*)ctx->pxy, (const float2*)ctx->pv, ctx->list, ns, ctx->ppart, de, (const uint64_t*)ctx->d_rg, ctx->d_rs,
                 (const uint64_t*)ctx->d_GS, (const uint8_t*)ctx->d_tflag, (const uint32_t*)ctx->d_gfx,
                 (const DevScalars*)ctx->sc, fc, par));
    if (int r = L_moments(ctx, st, ctx->d_GS, true)) return r;
    if (fork) CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    else if (int r = L_births(ctx, a, fc, st, nullptr, true, bl)) return r;
    ctx->k += 1;
    return DOG_OK;
}

// ---- row-band contexts: the cycle in four phases with the caller's exchanges in between
int dog_band_predict(dog_ctx* ctx, float dt, void* stream)
{
    if (!ctx) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world < 2 || ctx->phase != 0) return DOG_E_STATE;
    if (!(dt > 0.0f) || !finite(dt)) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    ctx->band_dt = dt;
    const StepArgs a = step_args(ctx, dt);
    const FilterConst fc = filter_const(ctx);
    CK(launch(k_predict_band, ctx->own_tiles, kPsThreads, 0, st, 0, (const float4*)ctx->st, ctx->pst, ctx->mg,
              ctx->sc, fc, a));
    CK(launch(k_pack_migrants, 1, 1024, 0, st, 0, ctx->mg, ctx->own_tiles, ctx->sc));
    ctx->phase = 1;
    return DOG_OK;
}

int dog_band_sizes(dog_ctx* ctx, uint32_t* counts, uint32_t* n_own, void* stream)
{
    if (!ctx || !counts || !n_own) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world < 2 || (ctx->phase != 1 && ctx->phase != 2)) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    DevScalars s;
    CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
    for (int d = 0; d < kMigDirs; ++d) counts[d] = s.mig_cnt[d];
    *n_own = s.n_own[ctx->k & 1];
    if (s.mig_over) {   // a bucket overflowed migrant_cap: the cycle cannot be completed exactly
        ctx->poisoned = true;
        return DOG_E_NOMEM;
    }
    return DOG_OK;
}

int dog_band_outbox(dog_ctx* ctx, const float** rec, const uint32_t** cnt)
{
    if (!ctx || !rec || !cnt) return DOG_E_INVAL;
    if (ctx->world < 2 || !ctx->shards.empty()) return DOG_E_STATE;
    for (int d = 0; d < kMigDirs; ++d) {
        rec[d] = (const float*)ctx->mg.send[d];
        cnt[d] = &ctx->sc->mig_cnt[d];
    }
    return DOG_OK;
}

int dog_band_gather(dog_ctx* ctx, const float* lo_near, const uint32_t* lo_near_cnt, const float* hi_near,
                    const uint32_t* hi_near_cnt, int n_lo_far, const float* const* lo_far,
                    const uint32_t* const* lo_far_cnt, int n_hi_far, const float* const* hi_far,
                    const uint32_t* const* hi_far_cnt, void* stream)
{
    if (!ctx) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world < 2 || ctx->phase != 1) return DOG_E_STATE;
    const int r = ctx->rank, w = ctx->world;
    if ((r > 0) != (lo_near != nullptr) || (r > 0 && !lo_near_cnt) || (r < w - 1) != (hi_near != nullptr) ||
        (r < w - 1 && !hi_near_cnt) || n_lo_far != std::max(0, r - 1) || n_hi_far != std::max(0, w - r - 2) ||
        (n_lo_far && (!lo_far || !lo_far_cnt)) || (n_hi_far && (!hi_far || !hi_far_cnt)))
        return DOG_E_INVAL;
    MigGather g{};
    g.lo_near = MigSrc{(const float4*)lo_near, lo_near_cnt};
    g.hi_near = MigSrc{(const float4*)hi_near, hi_near_cnt};
    g.n_lo_far = n_lo_far;
    g.n_hi_far = n_hi_far;
    for (int i = 0; i < n_lo_far; ++i) {
        if (!lo_far[i] || !lo_far_cnt[i]) return DOG_E_INVAL;
        g.lo_far[i] = MigSrc{(const float4*)lo_far[i], lo_far_cnt[i]};
    }
    for (int i = 0; i < n_hi_far; ++i) {
        if (!hi_far[i] || !hi_far_cnt[i]) return DOG_E_INVAL;
        g.hi_far[i] = MigSrc{(const float4*)hi_far[i], hi_far_cnt[i]};
    }
    if (int rc = set_device(ctx)) return rc;
    CK(launch(k_gather_migrants, 1 + 2 * 148, 1024, 0, (cudaStream_t)stream, 0, g, ctx->pst, ctx->sc,
              filter_const(ctx), ctx->own_cap + ctx->hi_cap, (int)(ctx->k & 1)));
    ctx->phase = 2;
    return DOG_OK;
}

int dog_band_assign(dog_ctx* ctx, const float* meas_band, const uint64_t** mass_dev, void* stream)
{
    if (!ctx || !meas_band || !mass_dev) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->phase != 2) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const StepArgs a = step_args(ctx, ctx->band_dt);
    const FilterConst fc = filter_const(ctx);
    if (int r = L_predict_sort(ctx, false, a, fc, st)) return r;
    if (int r = L_cells(ctx, meas_band, a, fc, st)) return r;
    *mass_dev = &ctx->sc->A_acc;
    ctx->phase = 3;
    return DOG_OK;
}

int dog_band_assign_exact(dog_ctx* ctx, const float* obs_band, const uint64_t** mass_dev, void* stream)
{
    if (!ctx || !obs_band || !mass_dev || ((uintptr_t)obs_band & 15u) != 0) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->phase != 2) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const StepArgs a = step_args(ctx, ctx->band_dt);
    const FilterConst fc = filter_const(ctx);
    if (int r = L_predict_sort(ctx, false, a, fc, st)) return r;
    if (int r = L_cells(ctx, nullptr, a, fc, st, obs_band)) return r;
    *mass_dev = &ctx->sc->A_acc;
    ctx->band_exact = true;
    ctx->phase = 3;
    return DOG_OK;
}

int dog_band_assign_doppler(dog_ctx* ctx, const float* meas_band, const float* doppler_band, const float* p_assoc_band,
                            const uint64_t** mass_dev, void* stream)
{
    if (!ctx || !doppler_band || !p_assoc_band || ((uintptr_t)doppler_band & 15u) != 0) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->phase != 2) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    if (int r = alloc_doppler(ctx)) return r;
    if (int r = dog_band_assign(ctx, meas_band, mass_dev, stream)) return r;
    // the per-run likelihood sums of the band's tiles (same kernel as the whole-grid branch)
    const StepArgs a = step_args(ctx, ctx->band_dt);
    const FilterConst fc = filter_const(ctx);
    const DopIn din{(const float4*)doppler_band, p_assoc_band};
    if (int r = L_dopp_runs(ctx, din, fc, (int)(a.k & 1), (cudaStream_t)stream)) return r;
    ctx->band_dop = doppler_band;
    ctx->band_pA = p_assoc_band;
    return DOG_OK;
}

int dog_band_joint(dog_ctx* ctx, const uint64_t* mass_all_dev, const uint64_t** weight_dev, void* stream)
{
    if (!ctx || !mass_all_dev || !weight_dev) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->phase != 3) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const StepArgs a = step_args(ctx, ctx->band_dt);
    const FilterConst fc = filter_const(ctx);
    if (int r = L_list_scan(ctx, mass_all_dev, a, fc, st, ctx->band_exact)) return r;
    *weight_dev = &ctx->sc->W;
    ctx->phase = 4;
    return DOG_OK;
}

int dog_band_resample(dog_ctx* ctx, const uint64_t* weight_all_dev, void* stream)
{
    if (!ctx || !weight_all_dev) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->phase != 4) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const StepArgs a = step_args(ctx, ctx->band_dt);
    const FilterConst fc = filter_const(ctx);
    if (ctx->band_pA) {   // Doppler cycle (dog_band_assign_doppler): as dog_step_doppler, on the band
        const DopIn din{(const float4*)ctx->band_dop, ctx->band_pA};
        const int par = (int)(a.k & 1);
        if (int r = L_pairs(ctx, weight_all_dev, a, fc, st, false, DopPS{ctx->band_pA, ctx->d_rg, ctx->d_GS, ctx->d_tflag, ctx->d_gmax}))
            return r;
        if (int r = L_resample(ctx, a, fc, st, ctx->d_GS)) return r;
        NextState ns{ctx->st, nullptr};
        CK(launch_ex(false, k_resample_dopp, ctx->tiles, 256, kRdSmemBytes, st, 0, ctx->tp,
                     (const float2*)ctx->pxy, (const float2*)ctx->pv, ctx->list, ns, ctx->ppart, din, (const uint64_t*)ctx->d_rg, ctx->d_rs,
                     (const uint64_t*)ctx->d_GS, (const uint8_t*)ctx->d_tflag, (const uint32_t*)ctx->d_gfx,
                     (const DevScalars*)ctx->sc, fc, par));
        if (int r = L_moments(ctx, st, ctx->d_GS)) return r;
        if (int r = L_births(ctx, a, fc, st, &din)) return r;
        ctx->band_dop = nullptr;
        ctx->band_pA = nullptr;
    } else {
        const bool ex = ctx->band_exact;          // exact filter: long lists, births in every cell
        if (int r = L_pairs(ctx, weight_all_dev, a, fc, st, ex)) return r;
        if (int r = L_resample(ctx, a, fc, st, nullptr, ex)) return r;
        if (int r = L_moments(ctx, st, nullptr, ex)) return r;
        if (int r = L_births(ctx, a, fc, st, nullptr, ex)) return r;
        ctx->band_exact = false;
    }
    ctx->phase = 0;
    ctx->k += 1;
    return DOG_OK;
}

int dog_band_particles(dog_ctx* ctx, float* xyvv_host, uint64_t cap, uint32_t* n_own, uint64_t* global_first)
{
    if (!ctx || !n_own) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    CK(cudaDeviceSynchronize());
    DevScalars s;
    CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
    const int par = (int)(ctx->k & 1);
    *n_own = s.n_own[par];
    if (global_first) *global_first = s.o_base[par];
    if (xyvv_host) {
        if (cap < *n_own) return DOG_E_INVAL;
        if (*n_own) CK(cudaMemcpy(xyvv_host, ctx->st + ctx->lo_cap, (size_t)*n_own * 16, cudaMemcpyDeviceToHost));
    }
    return DOG_OK;   // measurement flags are reported by dog_read_cells / dog_sync (not here: rebalancing
                     // calls this on every band and must not fail on one of them alone)
}

int dog_band_set_state(dog_ctx* ctx, const float* xyvv_host, uint32_t n_own, uint64_t global_first,
                       const float* m_free_host, float w_bar, int64_t k)
{
    if (!ctx || (n_own && !xyvv_host) || !m_free_host || !(w_bar >= 0.0f) || !finite(w_bar) || k < 0)
        return DOG_E_INVAL;
    if (ctx->world < 2) return DOG_E_STATE;
    if (ctx->phase != 0) return DOG_E_STATE;
    if (n_own > ctx->own_cap) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    CK(cudaDeviceSynchronize());
    const int par = (int)(k & 1);
    if (n_own) CK(cudaMemcpy(ctx->st + ctx->lo_cap, xyvv_host, (size_t)n_own * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->m_free, m_free_host, (size_t)ctx->C * 4, cudaMemcpyHostToDevice));
    DevScalars s;
    CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
    s.w_bar = w_bar;
    s.n_own[par] = n_own;
    s.o_base[par] = global_first;
    s.n_lo = 0; s.n_hi = 0;
    CK(cudaMemcpy(ctx->sc, &s, sizeof(s), cudaMemcpyHostToDevice));
    ctx->k = k;
    return DOG_OK;
}

int dog_profile_begin(dog_ctx* ctx, int max_steps)
{
    if (!ctx || max_steps < 0) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    for (cudaEvent_t e : ctx->pev) cudaEventDestroy(e);
    ctx->pev.assign((size_t)max_steps * (DOG_MAX_STAGES + 1), nullptr);
    for (auto& e : ctx->pev) CK(cudaEventCreate(&e));
    ctx->prof_max = max_steps;
    ctx->prof_steps = 0;
    return DOG_OK;
}

int dog_profile_end(dog_ctx* ctx, float* stage_ms, int* n_stages, int* n_steps)
{
    if (!ctx) return DOG_E_INVAL;
    if (int r = set_device(ctx)) return r;
    if (stage_ms)
        for (int i = 0; i < DOG_MAX_STAGES; ++i) stage_ms[i] = 0.0f;
    for (int s = 0; s < ctx->prof_steps; ++s) {
        cudaEvent_t* ev = &ctx->pev[(size_t)s * (DOG_MAX_STAGES + 1)];
        CK(cudaEventSynchronize(ev[ctx->prof_nst]));
        for (int i = 0; i < ctx->prof_nst; ++i) {
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            if (stage_ms) stage_ms[i] += ms;
        }
    }
    if (n_stages) *n_stages = ctx->prof_nst;
    if (n_steps) *n_steps = ctx->prof_steps;
    for (cudaEvent_t e : ctx->pev) cudaEventDestroy(e);
    ctx->pev.clear();
    ctx->prof_max = 0;
    ctx->prof_steps = 0;
    return DOG_OK;
}

const char* dog_profile_stage_name(dog_ctx* ctx, int i)
{
    if (!ctx || i < 0 || i >= DOG_MAX_STAGES || !ctx->stage_names[i]) return "";
    return ctx->stage_names[i];
}

int dog_step_host(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, void* stream)
{
    if (!ctx || !meas_host) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    if (!ctx->meas_dev) {
        int rc = dalloc(ctx, &ctx->meas_dev, 2 * (size_t)ctx->C);
        if (rc) return rc;
    }
    CK(cudaMemcpyAsync(ctx->meas_dev, meas_host, 8 * (size_t)ctx->C, cudaMemcpyHostToDevice, st));
    int rc = dog_step(ctx, ctx->meas_dev, dt, stream);
    if (rc) return rc;
    if (occ_host) CK(cudaMemcpyAsync(occ_host, ctx->occ, 4 * (size_t)ctx->C, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return DOG_OK;
}

static int step_host_pipelined(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, float* free_host,
                               float* mean_host, float* cov_host, void* stream)
{
    if (!ctx || !meas_host) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t C = ctx->C;
    if (!ctx->h2d) {   // first use: staging buffers (meas; the 7 readout floats per cell), copy streams, events
        for (int b = 0; b < 2; ++b) {
            if (int rc = dalloc(ctx, &ctx->hmeas[b], 2 * C)) return rc;
            if (int rc = dalloc(ctx, &ctx->hocc[b], 7 * C)) return rc;
            CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_used[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_out[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_read[b], cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->ev_used[b], st));
            CK(cudaEventRecord(ctx->ev_read[b], st));
        }
        CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    }
    const int b = ctx->hbuf;
    ctx->hbuf ^= 1;
    // in: wait until the cycle that last read this staging buffer is done, then copy the frame
    CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_used[b], 0));
    CK(cudaMemcpyAsync(ctx->hmeas[b], meas_host, 8 * C, cudaMemcpyHostToDevice, ctx->h2d));
    CK(cudaEventRecord(ctx->ev_in[b], ctx->h2d));
    // the cycle, on the caller's stream, once its frame has landed
    CK(cudaStreamWaitEvent(st, ctx->ev_in[b], 0));
    if (int rc = dog_step(ctx, ctx->hmeas[b], dt, stream)) return rc;
    CK(cudaEventRecord(ctx->ev_used[b], st));
    if (occ_host || free_host || mean_host || cov_host) {
        // out: snapshot the readouts on the device, copy them to the host while the next cycle runs
        float* snap = ctx->hocc[b];
        CK(cudaStreamWaitEvent(st, ctx->ev_read[b], 0));
        if (occ_host) CK(cudaMemcpyAsync(snap, ctx->occ, 4 * C, cudaMemcpyDeviceToDevice, st));
        if (free_host) CK(cudaMemcpyAsync(snap + C, ctx->fre, 4 * C, cudaMemcpyDeviceToDevice, st));
        if (mean_host) CK(cudaMemcpyAsync(snap + 2 * C, ctx->mean, 8 * C, cudaMemcpyDeviceToDevice, st));
        if (cov_host) CK(cudaMemcpyAsync(snap + 4 * C, ctx->cov, 12 * C, cudaMemcpyDeviceToDevice, st));
        CK(cudaEventRecord(ctx->ev_out[b], st));
        CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_out[b], 0));
        if (occ_host) CK(cudaMemcpyAsync(occ_host, snap, 4 * C, cudaMemcpyDeviceToHost, ctx->d2h));
        if (free_host) CK(cudaMemcpyAsync(free_host, snap + C, 4 * C, cudaMemcpyDeviceToHost, ctx->d2h));
        if (mean_host) CK(cudaMemcpyAsync(mean_host, snap + 2 * C, 8 * C, cudaMemcpyDeviceToHost, ctx->d2h));
        if (cov_host) CK(cudaMemcpyAsync(cov_host, snap + 4 * C, 12 * C, cudaMemcpyDeviceToHost, ctx->d2h));
        CK(cudaEventRecord(ctx->ev_read[b], ctx->d2h));
    }
    return DOG_OK;
}

int dog_step_host_async(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, void* stream)
{
    return step_host_pipelined(ctx, meas_host, dt, occ_host, nullptr, nullptr, nullptr, stream);
}

int dog_step_host_readout(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, float* free_host,
                          float* mean_host, float* cov_host, void* stream)
{
    return step_host_pipelined(ctx, meas_host, dt, occ_host, free_host, mean_host, cov_host, stream);
}

int dog_ego_scroll(dog_ctx* ctx, double dx, double dy, int32_t* shift_x, int32_t* shift_y, void* stream)
{
    if (!ctx || !std::isfinite(dx) || !std::isfinite(dy)) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1) return DOG_E_STATE;                 // whole-grid contexts only
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    // integer-cell part of (delta + residual), fp64 truncation toward zero; the fraction is kept (A-32)
    const double cs = (double)ctx->grid.cell_size;
    const double tx = dx + ctx->res_x, ty = dy + ctx->res_y;
    const double qx = std::trunc(tx / cs), qy = std::trunc(ty / cs);
    const int32_t W = ctx->grid.width, H = ctx->grid.height;
    if (!(std::fabs(qx) * 2.0 < (double)W) || !(std::fabs(qy) * 2.0 < (double)H)) return DOG_E_INVAL;
    const int32_t sx = (int32_t)qx, sy = (int32_t)qy;
    ctx->res_x = tx - qx * cs;
    ctx->res_y = ty - qy * cs;
    ctx->org_x -= qx * cs;                                  // the grid moves by -shift in the world
    ctx->org_y -= qy * cs;
    if (shift_x) *shift_x = sx;
    if (shift_y) *shift_y = sy;
    if (sx == 0 && sy == 0) return DOG_OK;
    const uint32_t sms = ctx->flat_blocks / 4u;
    CK(launch_ex(false, k_ego_grid, 8u * (uint32_t)sms, 256, 0, st, 0, (const float*)ctx->m_free, ctx->m_free_tmp,
                 sx, sy, W, H));
    CK(launch_ex(false, k_ego_particles, 8u * (uint32_t)sms, 256, 0, st, 0, ctx->st, (uint32_t)ctx->nu, sx, sy, W, H));
    std::swap(ctx->m_free, ctx->m_free_tmp);
    return DOG_OK;
}

int dog_get_origin(dog_ctx* ctx, double* origin_x, double* origin_y)
{
    if (!ctx) return DOG_E_INVAL;
    if (origin_x) *origin_x = ctx->org_x;
    if (origin_y) *origin_y = ctx->org_y;
    return DOG_OK;
}

int dog_eval_cells(dog_ctx* ctx, const float* mean_dev, const float* cov_dev, const uint8_t* valid_dev, int valid_mode,
                   const uint8_t* labels_dev, const uint8_t* mask_dev, const float* thr_host, int n_thr,
                   float* m_dev, uint64_t* counts_host, double* sums_host, void* stream)
{
    if (!ctx || n_thr < 0 || n_thr > kEvalMaxThr || (n_thr && !thr_host) || (valid_mode != 0 && valid_mode != 1))
        return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const float2* mean = mean_dev ? (const float2*)mean_dev : ctx->mean;   // NULL: the filter's readouts
    const float* cov = cov_dev ? cov_dev : ctx->cov;
    EvalThr thr{};
    int n_sorted = 0;
    {   // stable ascending sort of the non-NaN thresholds (-0 as +0); pos[t] = sorted position (-1: NaN)
        int idx[kEvalMaxThr];
        for (int t = 0; t < n_thr; ++t) { thr.pos[t] = -1; if (thr_host[t] == thr_host[t]) idx[n_sorted++] = t; }
        std::stable_sort(idx, idx + n_sorted, [&](int a, int b) { return thr_host[a] < thr_host[b]; });
        for (int p = 0; p < n_sorted; ++p) {
            const float v = thr_host[idx[p]];
            thr.v[p] = v == 0.f ? 0.f : v;
            thr.pos[idx[p]] = (int8_t)p;
        }
        // tab[b] = #{sorted thresholds with key < b 2^(32-bits)} (keys nondecreasing along the sorted list)
        int j = 0;
        for (int bkt = 0; bkt <= kEvBuckets; ++bkt) {
            const uint64_t lo = (uint64_t)bkt << (32 - kEvBucketBits);
            while (j < n_sorted && (uint64_t)eval_key(thr.v[j]) < lo) ++j;
            thr.tab[bkt] = (uint8_t)j;
        }
    }
    const uint32_t sms = ctx->flat_blocks / 4u;
    auto al = [](const void* p, uintptr_t a) { return ((uintptr_t)p % a) == 0; };
    const uint32_t* vbits = valid_mode == 1 ? (const uint32_t*)ctx->mvalid : (const uint32_t*)nullptr;
    const bool tma = !getenv("DOG_EVAL_NO_TMA") && al(mean, 16) && al(cov, 16) && al(valid_dev, 16) &&
                     al(labels_dev, 16) && al(mask_dev, 16) && ctx->C >= (uint32_t)kEvT;
    if (tma) {
        const uint32_t blocks = std::max<uint32_t>(1u, std::min<uint32_t>(2u * sms, ctx->C / kEvT));
        CK(launch_ex(false, k_eval_cells_tma, blocks, kEvThreads, kEvSmem, st, 0, mean, cov, valid_dev, vbits,
                     labels_dev, mask_dev, thr, n_thr, m_dev, ctx->ev_acc, ctx->ev_counts, ctx->ev_sums, ctx->C));
    } else {
        const uint32_t blocks = std::max<uint32_t>(1u, std::min<uint32_t>(8u * sms, (ctx->C + 255u) / 256u));
        CK(launch_ex(false, k_eval_cells, blocks, 256, 0, st, 0, mean, cov, valid_dev, vbits, labels_dev, mask_dev,
                     thr, n_thr, m_dev, ctx->ev_acc, ctx->ev_counts, ctx->ev_sums, ctx->C));
    }
    if (counts_host || sums_host) {
        if (counts_host) CK(cudaMemcpyAsync(counts_host, ctx->ev_counts, sizeof(uint64_t) * 4 * (size_t)n_thr,
                                            cudaMemcpyDeviceToHost, st));
        if (sums_host) CK(cudaMemcpyAsync(sums_host, ctx->ev_sums, sizeof(double) * 5, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return DOG_OK;
}

int dog_check_transforms(uint64_t* bad_host)
{
    if (!bad_host) return DOG_E_INVAL;
    unsigned long long* d = nullptr;
    const unsigned long long init[4] = {0ull, 0ull, 0ull, ~0ull};
    if (cudaMalloc(&d, sizeof(init)) != cudaSuccess) return DOG_E_NOMEM;
    cudaError_t e = cudaMemcpy(d, init, sizeof(init), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) { k_check_transforms<<<1184, 256>>>(d); e = cudaGetLastError(); }
    if (e == cudaSuccess) e = cudaMemcpy(bad_host, d, sizeof(init), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? DOG_OK : DOG_E_CUDA;
}

int dog_ego_residual(dog_ctx* ctx, double* rx, double* ry)
{
    if (!ctx) return DOG_E_INVAL;
    if (rx) *rx = ctx->res_x;
    if (ry) *ry = ctx->res_y;
    return DOG_OK;
}

static int sync_sharded(dog_ctx* ctx, void* stream);
static int read_cells_parent(dog_ctx* ctx, float* occ, float* free_mass, float* vel_mean, float* vel_cov, void* stream);
static int get_state_sharded(dog_ctx* ctx, float* x, float* y, float* vx, float* vy, float* w_bar, float* m_free,
                             int64_t* k);
static int set_state_sharded(dog_ctx* ctx, const float* x, const float* y, const float* vx, const float* vy,
                             float w_bar, const float* m_free, int64_t k);

int dog_sync(dog_ctx* ctx, void* stream)
{
    if (!ctx) return DOG_E_INVAL;
    if (!ctx->shards.empty()) return sync_sharded(ctx, stream);
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    if (ctx->d2h) CK(cudaStreamSynchronize(ctx->d2h));
    if (ctx->h2d) CK(cudaStreamSynchronize(ctx->h2d));
    return report_meas(ctx);
}

int dog_read_cells(dog_ctx* ctx, float* occ, float* free_mass, float* vel_mean, float* vel_cov, void* stream)
{
    if (!ctx) return DOG_E_INVAL;
    if (!ctx->shards.empty()) return read_cells_parent(ctx, occ, free_mass, vel_mean, vel_cov, stream);
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t C = ctx->C;
    if (occ) CK(cudaMemcpyAsync(occ, ctx->occ, 4 * C, cudaMemcpyDeviceToDevice, st));
    if (free_mass) CK(cudaMemcpyAsync(free_mass, ctx->fre, 4 * C, cudaMemcpyDeviceToDevice, st));
    if (vel_mean) CK(cudaMemcpyAsync(vel_mean, ctx->mean, 8 * C, cudaMemcpyDeviceToDevice, st));
    if (vel_cov) CK(cudaMemcpyAsync(vel_cov, ctx->cov, 12 * C, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return report_meas(ctx);
}

int dog_get_state(dog_ctx* ctx, float* x, float* y, float* vx, float* vy, float* w_bar, float* m_free,
                  int64_t* k)
{
    if (!ctx) return DOG_E_INVAL;
    if (!ctx->shards.empty()) return get_state_sharded(ctx, x, y, vx, vy, w_bar, m_free, k);
    if (ctx->world > 1 && (x || y || vx || vy)) return DOG_E_STATE;   // band particles: dog_band_particles
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    CK(cudaDeviceSynchronize());
    float* comp[4] = {x, y, vx, vy};
    for (int c = 0; c < 4; ++c)   // one component of the (x, y, vx, vy) records: strided copy
        if (comp[c]) CK(cudaMemcpy2D(comp[c], 4, (const float*)ctx->st + c, 16, 4, (size_t)ctx->nu, cudaMemcpyDeviceToHost));
    if (m_free) CK(cudaMemcpy(m_free, ctx->m_free, (size_t)ctx->C * 4, cudaMemcpyDeviceToHost));
    if (w_bar) CK(cudaMemcpy(w_bar, &ctx->sc->w_bar, 4, cudaMemcpyDeviceToHost));
    if (k) *k = ctx->k;
    return report_meas(ctx);
}

int dog_set_state(dog_ctx* ctx, const float* x, const float* y, const float* vx, const float* vy, float w_bar,
                  const float* m_free, int64_t k)
{
    if (!ctx || !x || !y || !vx || !vy || !m_free || !(w_bar >= 0.0f) || !finite(w_bar) || k < 0)
        return DOG_E_INVAL;
    if (!ctx->shards.empty()) return set_state_sharded(ctx, x, y, vx, vy, w_bar, m_free, k);
    if (ctx->world > 1) return DOG_E_STATE;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (int r = set_device(ctx)) return r;
    CK(cudaDeviceSynchronize());
    const float* comp[4] = {x, y, vx, vy};
    for (int c = 0; c < 4; ++c)
        CK(cudaMemcpy2D((float*)ctx->st + c, 16, comp[c], 4, 4, (size_t)ctx->nu, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->m_free, m_free, (size_t)ctx->C * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(&ctx->sc->w_bar, &w_bar, 4, cudaMemcpyHostToDevice));
    ctx->k = k;
    return DOG_OK;
}

int64_t dog_get_debug(dog_ctx* ctx, int what, void* host_dst, size_t bytes)
{
    if (!ctx || !host_dst) return DOG_E_INVAL;
    if (ctx->poisoned) return DOG_E_CUDA;
    if (ctx->world > 1 && what != DOG_DBG_SCALARS) return DOG_E_STATE;
    if (int r = set_device(ctx)) return r;
    CK(cudaDeviceSynchronize());
    const bool dbg = (ctx->flags & DOG_FLAG_DEBUG) != 0;
    const size_t nu = (size_t)ctx->nu, C = ctx->C, nb = (size_t)ctx->nu_b;
    const void* src = nullptr;
    size_t n = 0;
    // the flat active-cell list (for OFFSETS / NB reconstruction)
    auto read_list = [&](std::vector<uint32_t>& lc, std::vector<uint32_t>& ln, std::vector<uint32_t>& lst,
                         std::vector<uint32_t>& lnb, uint32_t& Ln, uint64_t& n_in) -> int {
        DevScalars s;
        CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
        n_in = s.n_in;
        Ln = s.Lc;
        lc.resize(Ln); ln.resize(Ln); lst.resize(Ln); lnb.resize(Ln);
        if (Ln) {
            CK(cudaMemcpy(lc.data(), ctx->list.c, (size_t)Ln * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(ln.data(), ctx->list.n, (size_t)Ln * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(lst.data(), ctx->list.start, (size_t)Ln * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(lnb.data(), ctx->list.nb, (size_t)Ln * 4, cudaMemcpyDeviceToHost));
        }
        return DOG_OK;
    };
    switch (what) {
    case DOG_DBG_PRED_X: case DOG_DBG_PRED_Y: case DOG_DBG_PRED_VX: case DOG_DBG_PRED_VY: {
        n = nu * 4;
        if (bytes < n) return DOG_E_INVAL;
        const int c = what - DOG_DBG_PRED_X;
        if (!dbg) return DOG_E_STATE;              // input-order predicted state: debug builds only
        CK(cudaMemcpy2D(host_dst, 4, (const float*)ctx->pst + c, 16, 4, nu, cudaMemcpyDeviceToHost));
        return (int64_t)n;
    }
    case DOG_DBG_KEY: if (!dbg) return DOG_E_STATE; src = ctx->keys; n = nu * 4; break;
    case DOG_DBG_PERM: {   // cell-sorted slots [0, n_in) from the resample kernel; sentinels follow in input order
        if (!dbg) return DOG_E_STATE;
        n = nu * 4;
        if (bytes < n) return DOG_E_INVAL;
        DevScalars s;
        CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
        uint32_t* dst = (uint32_t*)host_dst;
        if (s.n_in) CK(cudaMemcpy(dst, ctx->perm, s.n_in * 4, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> kk(nu);
        CK(cudaMemcpy(kk.data(), ctx->keys, nu * 4, cudaMemcpyDeviceToHost));
        size_t o = s.n_in;
        for (size_t i = 0; i < nu; ++i)
            if (kk[i] >= ctx->C) dst[o++] = (uint32_t)i;
        return (int64_t)n;
    }
    case DOG_DBG_RHO_P: if (!dbg) return DOG_E_STATE; src = ctx->dbg_rho_p; n = C * 4; break;
    case DOG_DBG_RHO_B: if (!dbg) return DOG_E_STATE; src = ctx->dbg_rho_b; n = C * 4; break;
    case DOG_DBG_RP: if (!dbg) return DOG_E_STATE; src = ctx->dbg_Rp; n = C * 8; break;
    case DOG_DBG_RB: if (!dbg) return DOG_E_STATE; src = ctx->dbg_Rb; n = C * 8; break;
    case DOG_DBG_BIRTH_X: if (!dbg) return DOG_E_STATE; src = ctx->bx; n = nb * 4; break;
    case DOG_DBG_BIRTH_Y: if (!dbg) return DOG_E_STATE; src = ctx->by; n = nb * 4; break;
    case DOG_DBG_BIRTH_VX: if (!dbg) return DOG_E_STATE; src = ctx->bvx; n = nb * 4; break;
    case DOG_DBG_BIRTH_VY: if (!dbg) return DOG_E_STATE; src = ctx->bvy; n = nb * 4; break;
    case DOG_DBG_JOINT_IDX: if (!dbg) return DOG_E_STATE; src = ctx->jidx; n = nu * 4; break;
    case DOG_DBG_OFFSETS: {
        n = (C + 1) * 4;
        if (bytes < n) return DOG_E_INVAL;
        std::vector<uint32_t> lc, ln, lst, lnb;
        uint32_t Ln; uint64_t n_in;
        if (int r = read_list(lc, ln, lst, lnb, Ln, n_in)) return r;
        uint32_t* d = (uint32_t*)host_dst;
        uint32_t next = (uint32_t)n_in;   // first sorted slot of the next cell holding particles
        int64_t li = (int64_t)Ln - 1;
        d[C] = (uint32_t)n_in;
        for (int64_t c = (int64_t)C - 1; c >= 0; --c) {
            while (li >= 0 && lc[li] > (uint32_t)c) --li;
            if (li >= 0 && lc[li] == (uint32_t)c && ln[li] > 0) next = lst[li];
            d[c] = next;
        }
        return (int64_t)n;
    }
    case DOG_DBG_NB: {
        n = C * 4;
        if (bytes < n) return DOG_E_INVAL;
        std::vector<uint32_t> lc, ln, lst, lnb;
        uint32_t Ln; uint64_t n_in;
        if (int r = read_list(lc, ln, lst, lnb, Ln, n_in)) return r;
        uint32_t* d = (uint32_t*)host_dst;
        for (size_t c = 0; c < C; ++c) d[c] = 0;
        for (uint32_t i = 0; i < Ln; ++i) d[lc[i]] = lnb[i];
        return (int64_t)n;
    }
    case DOG_DBG_SCALARS: {
        n = 8 * 8;
        if (bytes < n) return DOG_E_INVAL;
        DevScalars s;
        CK(cudaMemcpy(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost));
        uint64_t* d = (uint64_t*)host_dst;
        uint32_t wp, wb;
        memcpy(&wp, &s.w_pred, 4);
        memcpy(&wb, &s.w_bar, 4);
        d[0] = s.W; d[1] = s.U; d[2] = s.A; d[3] = s.meas_bad; d[4] = wp; d[5] = wb;
        d[6] = (uint64_t)(ctx->k - 1); d[7] = s.n_in;
        return (int64_t)n;
    }
    default: return DOG_E_INVAL;
    }
    if (bytes < n) return DOG_E_INVAL;
    if (n) CK(cudaMemcpy(host_dst, src, n, cudaMemcpyDeviceToHost));
    return (int64_t)n;
}


// ================================================================================================
// Sharded parent context: dog_create with n_devices >= 2 makes one
// row-band context per device (bottom-up bands of near-equal height).  dog_step_sharded runs the four
// band phases on every device and moves what the bands couple ENTIRELY ON THE DEVICES, ordered only by
// CUDA events: (1) the receivers' k_gather_migrants read the senders' packed migrant buckets and their
// device counts over peer memory (NVLink; the same memory when bands share a device), (2)/(3) a
// one-warp k_gather_u64 reads every band's born-mass / joint-weight total.  No host synchronisation
// inside a cycle.  Every band can hold all nu particles in each of its three regions (migrant_cap = nu),
// so a receive cannot overflow, and the owner-bucketed migration reaches any band: no particle is lost.
// ================================================================================================
struct U64Gather {
    const uint64_t* p[kMaxBands];
    int n;
};

__global__ void k_gather_u64(U64Gather g, uint64_t* __restrict__ out)
{
    PDL_ENTER();
    if ((int)threadIdx.x < g.n) out[threadIdx.x] = *g.p[threadIdx.x];
}

namespace {

struct DevGuard {   // restores the caller's current device
    int prev = -1;
    DevGuard() { cudaGetDevice(&prev); }
    ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

void destroy_shards(dog_ctx* P)
{
    for (size_t s = 0; s < P->shards.size(); ++s) {
        cudaSetDevice(P->shard_dev[s]);
        cudaDeviceSynchronize();
        for (auto* v : {&P->sev_pred, &P->sev_asg, &P->sev_jnt, &P->sev_done})
            if (s < v->size() && (*v)[s]) cudaEventDestroy((*v)[s]);
        if (s < P->shard_st.size() && P->shard_st[s]) cudaStreamDestroy(P->shard_st[s]);
        if (P->shards[s]) dog_destroy(P->shards[s]);
    }
    P->shards.clear();
    P->shard_st.clear();
    P->sev_pred.clear(); P->sev_asg.clear(); P->sev_jnt.clear(); P->sev_done.clear();
    P->sh_mass.clear(); P->sh_weight.clear();
}

// (re)create the band contexts of a parent on rows[0..world] (validated by the caller)
int make_shards(dog_ctx* P, const std::vector<int32_t>& rows)
{
    const int w = (int)P->shard_dev.size();
    P->shard_rows = rows;
    P->shards.assign(w, nullptr);
    P->shard_st.assign(w, nullptr);
    P->sev_pred.assign(w, nullptr); P->sev_asg.assign(w, nullptr); P->sev_jnt.assign(w, nullptr);
    P->sev_done.assign(w, nullptr);
    P->sh_mass.assign(w, nullptr); P->sh_weight.assign(w, nullptr);
    const uint32_t cap = (uint32_t)std::min<int64_t>(P->nu, (1 << 26) - 1);
    for (int s = 0; s < w; ++s) {
        if (cudaSetDevice(P->shard_dev[s]) != cudaSuccess) { cudaGetLastError(); return DOG_E_INVAL; }
        dog_band b{rows[s], rows[s + 1], s, w, s > 0 ? rows[s - 1] : rows[s], s < w - 1 ? rows[s + 2] : rows[s + 1], cap};
        if (int rc = create_impl(&P->grid, P->nu, P->nu_b, &P->params, P->seed, 0, &b, &P->shards[s])) return rc;
        dog_ctx* S = P->shards[s];
        int rc = dalloc(S, &P->sh_mass[s], (size_t)w);
        if (rc == DOG_OK) rc = dalloc(S, &P->sh_weight[s], (size_t)w);
        if (rc) return rc;
        for (auto* v : {&P->sev_pred, &P->sev_asg, &P->sev_jnt, &P->sev_done})
            if (cudaEventCreateWithFlags(&(*v)[s], cudaEventDisableTiming) != cudaSuccess) return fail(P, cudaGetLastError(), "cudaEventCreate");
        if (cudaStreamCreateWithFlags(&P->shard_st[s], cudaStreamNonBlocking) != cudaSuccess)
            return fail(P, cudaGetLastError(), "cudaStreamCreate");
    }
    return DOG_OK;
}

std::vector<int32_t> even_rows(int32_t H, int w)
{
    std::vector<int32_t> r(w + 1, 0);
    const int32_t base = H / w, extra = H % w;
    for (int s = 0; s < w; ++s) r[s + 1] = r[s] + base + (s < extra ? 1 : 0);
    return r;
}

bool rows_valid(const int32_t* rows, int w, int32_t H)
{
    if (rows[0] != 0 || rows[w] != H) return false;
    for (int s = 0; s < w; ++s)
        if (rows[s + 1] <= rows[s]) return false;
    return true;
}

// one band of the cycle: phase `ph` (0 predict, 1 gather + assign, 2 totals + joint, 3 totals + resample)
int shard_phase(dog_ctx* P, int s, int ph, const float* meas_band, float dt, cudaStream_t st)
{
    dog_ctx* S = P->shards[s];
    const int w = (int)P->shards.size();
    if (cudaSetDevice(P->shard_dev[s]) != cudaSuccess) return fail(P, cudaGetLastError(), "cudaSetDevice");
    auto wait_all = [&](std::vector<cudaEvent_t>& ev) -> int {
        for (int t = 0; t < w; ++t)
            if (t != s) CK2(P, cudaStreamWaitEvent(st, ev[t], 0));
        return DOG_OK;
    };
    int rc = DOG_OK;
    switch (ph) {
    case 0:
        rc = dog_band_predict(S, dt, st);
        if (!rc) CK2(P, cudaEventRecord(P->sev_pred[s], st));
        return rc;
    case 1: {
        if (int r = wait_all(P->sev_pred)) return r;
        const float* rec[kMaxBands][kMigDirs];
        const uint32_t* cnt[kMaxBands][kMigDirs];
        for (int t = 0; t < w; ++t) dog_band_outbox(P->shards[t], rec[t], cnt[t]);
        const float* lof[kMaxBands]; const uint32_t* lofc[kMaxBands];
        const float* hif[kMaxBands]; const uint32_t* hifc[kMaxBands];
        int nl = 0, nh = 0;
        for (int t = 0; t < s - 1; ++t) { lof[nl] = rec[t][3]; lofc[nl++] = cnt[t][3]; }
        for (int t = s + 2; t < w; ++t) { hif[nh] = rec[t][2]; hifc[nh++] = cnt[t][2]; }
        rc = dog_band_gather(S, s > 0 ? rec[s - 1][1] : nullptr, s > 0 ? cnt[s - 1][1] : nullptr,
                             s < w - 1 ? rec[s + 1][0] : nullptr, s < w - 1 ? cnt[s + 1][0] : nullptr,
                             nl, lof, lofc, nh, hif, hifc, st);
        const uint64_t* mass = nullptr;
        if (!rc) rc = dog_band_assign(S, meas_band, &mass, st);
        if (!rc) CK2(P, cudaEventRecord(P->sev_asg[s], st));
        return rc;
    }
    case 2:
    case 3: {
        if (int r = wait_all(ph == 2 ? P->sev_asg : P->sev_jnt)) return r;
        U64Gather g{};
        g.n = w;
        for (int t = 0; t < w; ++t) g.p[t] = ph == 2 ? &P->shards[t]->sc->A_acc : &P->shards[t]->sc->W;
        uint64_t* dst = ph == 2 ? P->sh_mass[s] : P->sh_weight[s];
        CK2(P, launch(k_gather_u64, 1, 32, 0, st, 0, g, dst));
        if (ph == 2) {
            const uint64_t* wd = nullptr;
            rc = dog_band_joint(S, dst, &wd, st);
            if (!rc) CK2(P, cudaEventRecord(P->sev_jnt[s], st));
        } else {
            rc = dog_band_resample(S, dst, st);
        }
        return rc;
    }
    }
    return DOG_E_INVAL;
}

int sharded_cycle(dog_ctx* P, const float* const* meas_band, float dt, const cudaStream_t* st)
{
    if (P->poisoned) return DOG_E_CUDA;
    if (!(dt > 0.0f) || !finite(dt)) return DOG_E_INVAL;
    const int w = (int)P->shards.size();
    for (int ph = 0; ph < 4; ++ph)
        for (int s = 0; s < w; ++s)
            if (int rc = shard_phase(P, s, ph, meas_band[s], dt, st[s])) {
                P->poisoned = true;   // bands are mid-cycle: only dog_destroy
                return rc;
            }
    P->k += 1;
    return DOG_OK;
}

}  // namespace

static int create_sharded(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
                          uint64_t seed, uint32_t flags, int n_devices, const int* device_ids, dog_ctx** out)
{
    if (!grid || !params || n_devices > kMaxBands || (flags & DOG_FLAG_DEBUG)) return DOG_E_INVAL;
    if (grid->height < n_devices) return DOG_E_INVAL;
    *out = nullptr;
    DevGuard guard;
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int s = 0; s < n_devices; ++s)
        if (device_ids[s] < 0 || device_ids[s] >= ndev) return DOG_E_INVAL;
    // peer access between every pair of distinct devices (NVLink / NVSwitch); required
    for (int a = 0; a < n_devices; ++a)
        for (int b = 0; b < n_devices; ++b) {
            const int da = device_ids[a], db = device_ids[b];
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) return DOG_E_INVAL;
            cudaSetDevice(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(nullptr, e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    dog_ctx* P = new (std::nothrow) dog_ctx();
    if (!P) return DOG_E_NOMEM;
    P->device = device_ids[0];
    P->grid = *grid;
    P->org_x = (double)grid->origin_x;
    P->org_y = (double)grid->origin_y;
    P->params = *params;
    P->seed = seed;
    P->nu = n_particles;
    P->nu_b = n_birth;
    P->Cg = (uint32_t)((int64_t)grid->width * grid->height);
    P->C = P->Cg;
    P->world = n_devices;
    P->shard_dev.assign(device_ids, device_ids + n_devices);
    int rc = make_shards(P, even_rows(grid->height, n_devices));
    if (rc == DOG_OK) {
        cudaSetDevice(device_ids[0]);
        if (cudaEventCreateWithFlags(&P->ev_caller, cudaEventDisableTiming) != cudaSuccess) rc = DOG_E_CUDA;
    }
    if (rc != DOG_OK) {
        destroy_shards(P);
        delete P;
        return rc;
    }
    *out = P;
    return DOG_OK;
}

static int destroy_sharded(dog_ctx* P)
{
    DevGuard guard;
    destroy_shards(P);
    if (P->ev_caller) { cudaSetDevice(P->device); cudaEventDestroy(P->ev_caller); }
    delete P;
    return DOG_OK;
}

int dog_world(dog_ctx* ctx)
{
    if (!ctx) return DOG_E_INVAL;
    return ctx->shards.empty() ? 1 : (int)ctx->shards.size();
}

int dog_get_bands(dog_ctx* ctx, int32_t* rows, int* devices)
{
    if (!ctx || !rows) return DOG_E_INVAL;
    if (ctx->shards.empty()) {
        rows[0] = 0; rows[1] = ctx->grid.height;
        if (devices) devices[0] = ctx->device;
        return 1;
    }
    for (size_t s = 0; s <= ctx->shards.size(); ++s) rows[s] = ctx->shard_rows[s];
    if (devices)
        for (size_t s = 0; s < ctx->shards.size(); ++s) devices[s] = ctx->shard_dev[s];
    return (int)ctx->shards.size();
}

int dog_step_sharded(dog_ctx* ctx, const float* const* meas_band, float dt, void* const* streams)
{
    if (!ctx || !meas_band || !streams) return DOG_E_INVAL;
    if (ctx->shards.empty()) return DOG_E_STATE;
    const int w = (int)ctx->shards.size();
    for (int s = 0; s < w; ++s)
        if (!meas_band[s]) return DOG_E_INVAL;
    DevGuard guard;
    std::vector<cudaStream_t> st(w);
    for (int s = 0; s < w; ++s) st[s] = (cudaStream_t)streams[s];
    return sharded_cycle(ctx, meas_band, dt, st.data());
}

int dog_read_cells_sharded(dog_ctx* ctx, float* const* occ, float* const* free_mass, float* const* vel_mean,
                           float* const* vel_cov, void* const* streams)
{
    if (!ctx || !streams) return DOG_E_INVAL;
    if (ctx->shards.empty()) return DOG_E_STATE;
    if (ctx->poisoned) return DOG_E_CUDA;
    DevGuard guard;
    int first = DOG_OK;
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const int rc = dog_read_cells(ctx->shards[s], occ ? occ[s] : nullptr, free_mass ? free_mass[s] : nullptr,
                                      vel_mean ? vel_mean[s] : nullptr, vel_cov ? vel_cov[s] : nullptr, streams[s]);
        if (rc && !first) first = rc;
    }
    return first;
}

int dog_set_bands(dog_ctx* ctx, const int32_t* rows)
{
    if (!ctx || !rows) return DOG_E_INVAL;
    if (ctx->shards.empty()) return DOG_E_STATE;
    if (ctx->poisoned) return DOG_E_CUDA;
    const int w = (int)ctx->shards.size();
    if (!rows_valid(rows, w, ctx->grid.height)) return DOG_E_INVAL;
    const size_t nu = (size_t)ctx->nu, C = ctx->Cg;
    std::vector<float> x(nu), y(nu), vx(nu), vy(nu), mf(C);
    float wb = 0.0f;
    int64_t k = 0;
    if (int rc = get_state_sharded(ctx, x.data(), y.data(), vx.data(), vy.data(), &wb, mf.data(), &k)) return rc;
    DevGuard guard;
    destroy_shards(ctx);
    if (int rc = make_shards(ctx, std::vector<int32_t>(rows, rows + w + 1))) {
        ctx->poisoned = true;
        return rc;
    }
    return set_state_sharded(ctx, x.data(), y.data(), vx.data(), vy.data(), wb, mf.data(), k);
}

static int step_parent(dog_ctx* P, const float* meas, float dt, void* stream)
{
    // meas on device_ids[0] (peer-readable by every band); the bands run on the parent's own streams,
    // forked from and joined back into the caller's stream
    if (P->poisoned) return DOG_E_CUDA;
    DevGuard guard;
    const int w = (int)P->shards.size();
    cudaSetDevice(P->device);
    CK2(P, cudaEventRecord(P->ev_caller, (cudaStream_t)stream));
    std::vector<const float*> mb(w);
    for (int s = 0; s < w; ++s) {
        cudaSetDevice(P->shard_dev[s]);
        CK2(P, cudaStreamWaitEvent(P->shard_st[s], P->ev_caller, 0));
        mb[s] = meas + (size_t)P->shard_rows[s] * P->grid.width * 2;
    }
    if (int rc = sharded_cycle(P, mb.data(), dt, P->shard_st.data())) return rc;
    for (int s = 0; s < w; ++s) {
        cudaSetDevice(P->shard_dev[s]);
        CK2(P, cudaEventRecord(P->sev_done[s], P->shard_st[s]));
    }
    cudaSetDevice(P->device);
    for (int s = 0; s < w; ++s) CK2(P, cudaStreamWaitEvent((cudaStream_t)stream, P->sev_done[s], 0));
    return DOG_OK;
}

static int sync_sharded(dog_ctx* P, void* stream)
{
    if (P->poisoned) return DOG_E_CUDA;
    DevGuard guard;
    cudaSetDevice(P->device);
    CK2(P, cudaStreamSynchronize((cudaStream_t)stream));
    int first = DOG_OK;
    for (size_t s = 0; s < P->shards.size(); ++s) {
        cudaSetDevice(P->shard_dev[s]);
        CK2(P, cudaDeviceSynchronize());
        const int rc = report_meas(P->shards[s]);
        if (rc && !first) first = rc;
        if (P->shards[s]->poisoned) P->poisoned = true;
    }
    return first;
}

static int read_cells_parent(dog_ctx* P, float* occ, float* free_mass, float* vel_mean, float* vel_cov, void* stream)
{
    // whole-grid outputs on device_ids[0]: each band's rows copied peer-to-peer at its row offset
    if (P->poisoned) return DOG_E_CUDA;
    DevGuard guard;
    int first = DOG_OK;
    for (size_t s = 0; s < P->shards.size(); ++s) {   // the bands' cycles must be complete
        cudaSetDevice(P->shard_dev[s]);
        CK2(P, cudaDeviceSynchronize());
    }
    cudaSetDevice(P->device);
    cudaStream_t st = (cudaStream_t)stream;
    for (size_t s = 0; s < P->shards.size(); ++s) {
        dog_ctx* S = P->shards[s];
        const size_t off = (size_t)P->shard_rows[s] * P->grid.width, n = S->C;
        const int d = P->shard_dev[s];
        if (occ) CK2(P, cudaMemcpyPeerAsync(occ + off, P->device, S->occ, d, 4 * n, st));
        if (free_mass) CK2(P, cudaMemcpyPeerAsync(free_mass + off, P->device, S->fre, d, 4 * n, st));
        if (vel_mean) CK2(P, cudaMemcpyPeerAsync(vel_mean + 2 * off, P->device, S->mean, d, 8 * n, st));
        if (vel_cov) CK2(P, cudaMemcpyPeerAsync(vel_cov + 3 * off, P->device, S->cov, d, 12 * n, st));
    }
    CK2(P, cudaStreamSynchronize(st));
    for (size_t s = 0; s < P->shards.size(); ++s) {
        cudaSetDevice(P->shard_dev[s]);
        const int rc = report_meas(P->shards[s]);
        if (rc && !first) first = rc;
    }
    return first;
}

static int get_state_sharded(dog_ctx* P, float* x, float* y, float* vx, float* vy, float* w_bar, float* m_free,
                             int64_t* k)
{
    // the bands' own particles in band (= global index) order; the empty remainder is sentinel particles
    // (the whole-grid state's particles outside the grid: they carry no weight and are never resampled)
    if (P->poisoned) return DOG_E_CUDA;
    DevGuard guard;
    const size_t nu = (size_t)P->nu;
    std::vector<float> rec;
    size_t n_tot = 0;
    for (size_t s = 0; s < P->shards.size(); ++s) {
        dog_ctx* S = P->shards[s];
        uint32_t n = 0;
        uint64_t g0 = 0;
        if (int rc = dog_band_particles(S, nullptr, 0, &n, &g0)) return rc;
        if (n_tot + n > nu) return DOG_E_STATE;
        rec.resize((size_t)n * 4);
        if (n) {
            if (int rc = dog_band_particles(S, rec.data(), n, &n, &g0)) return rc;
            if (g0 != n_tot) return DOG_E_STATE;     // bands are contiguous in global index order
        }
        for (uint32_t i = 0; i < n; ++i) {
            if (x) x[n_tot + i] = rec[4 * i];
            if (y) y[n_tot + i] = rec[4 * i + 1];
            if (vx) vx[n_tot + i] = rec[4 * i + 2];
            if (vy) vy[n_tot + i] = rec[4 * i + 3];
        }
        n_tot += n;
        if (m_free) {
            cudaSetDevice(P->shard_dev[s]);
            CK2(P, cudaMemcpy(m_free + (size_t)P->shard_rows[s] * P->grid.width, S->m_free, (size_t)S->C * 4,
                              cudaMemcpyDeviceToHost));
        }
    }
    for (size_t i = n_tot; i < nu; ++i) {
        if (x) x[i] = kSentinelPos;
        if (y) y[i] = kSentinelPos;
        if (vx) vx[i] = 0.0f;
        if (vy) vy[i] = 0.0f;
    }
    if (w_bar) {
        cudaSetDevice(P->shard_dev[0]);
        CK2(P, cudaMemcpy(w_bar, &P->shards[0]->sc->w_bar, 4, cudaMemcpyDeviceToHost));
    }
    if (k) *k = P->k;
    return DOG_OK;
}

static int set_state_sharded(dog_ctx* P, const float* x, const float* y, const float* vx, const float* vy,
                             float w_bar, const float* m_free, int64_t k)
{
    // each band's particles must be one contiguous range of the canonical order, ranges in band order;
    // particles outside the grid belong to no band (they carry no weight) and may sit anywhere else
    if (P->poisoned) return DOG_E_CUDA;
    const int w = (int)P->shards.size();
    const size_t nu = (size_t)P->nu;
    const float Wf = (float)P->grid.width, Hf = (float)P->grid.height;
    std::vector<int64_t> first(w, -1), last(w, -1);
    int prev_band = -1;
    for (size_t i = 0; i < nu; ++i) {
        const bool inside = x[i] >= 0.0f && x[i] < Wf && y[i] >= 0.0f && y[i] < Hf;
        if (!inside) continue;
        const int32_t row = (int32_t)y[i];
        int b = 0;
        while (row >= P->shard_rows[b + 1]) ++b;
        if (b < prev_band) return DOG_E_INVAL;
        if (first[b] < 0) first[b] = (int64_t)i;
        else if (last[b] != (int64_t)i - 1) return DOG_E_INVAL;   // a particle outside the grid splits the band
        last[b] = (int64_t)i;
        prev_band = b;
    }
    DevGuard guard;
    std::vector<float> rec;
    for (int b = 0; b < w; ++b) {
        const size_t n = first[b] < 0 ? 0 : (size_t)(last[b] - first[b] + 1);
        const size_t f0 = first[b] < 0 ? 0 : (size_t)first[b];
        rec.resize(4 * n + 4);
        for (size_t i = 0; i < n; ++i) {
            rec[4 * i] = x[f0 + i]; rec[4 * i + 1] = y[f0 + i]; rec[4 * i + 2] = vx[f0 + i]; rec[4 * i + 3] = vy[f0 + i];
        }
        const size_t off = (size_t)P->shard_rows[b] * P->grid.width;
        if (int rc = dog_band_set_state(P->shards[b], n ? rec.data() : nullptr, (uint32_t)n, f0, m_free + off, w_bar, k))
            return rc;
    }
    P->k = k;
    return DOG_OK;
}

#ifdef DOG_TIMING
int dog_timing_dump(unsigned long long* host, int n, int reset)
{
    if (cudaMemcpyFromSymbol(host, g_phase_ns, (size_t)n * 8) != cudaSuccess) return -1;
    if (reset) {
        static unsigned long long z[64] = {};
        cudaMemcpyToSymbol(g_phase_ns, z, sizeof(z));
    }
    return 0;
}
#endif

}  // extern "C"
