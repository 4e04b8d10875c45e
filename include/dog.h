/*
 * dog.h -- C ABI of the B200-native DS-PHD/MIB dynamic occupancy grid filter (libdog.so).
 *
 * One call of dog_step runs one full filter cycle k -> k+1 of the particle-based DS-PHD/MIB filter
 * of Nuss et al., arXiv 1605.02406 (section VI; parallel pipeline section VII,
 * P:1249-1520) on the GPU, with a measurement grid of occupied/free masses only (spatial likelihood
 * g = 1, association probability p_A = 0, Abar birth set only; A-27):
 *   1 predict      CV model x' = F(T) x + xi (Eq. 14), w = p_S w (Eq. 39)
 *   2 assign       stable sort of particles by cell key, per-cell offsets (Alg. 2)
 *   3 cells        m_p = min(sum w, occ_max) (Eqs. 17/61), m_Fp = min(alpha m_F, 1 - m_p) (Eq. 62),
 *                  (m_O, m_F) = Dempster(m_p, meas) (Eq. 63), birth split rho_b/rho_p (Eqs. 67-68)
 *   4 persistent   w = rho_p / m_p * w_pred (Eq. 71 with p_A = 0, Eq. 73)
 *   5 births       nu_b new particles in proportion to rho_b (Alg. 5)
 *   6 moments      per-cell velocity mean / covariance of persistent particles (Eqs. 81-84)
 *   7 resample     systematic resampling to nu particles of equal weight (Alg. 7, Eq. 57)
 *
 * Conventions:
 *   - grid: width x height cells, x = column (fastest), y = row; cell key c = row*width + col.
 *     Particle positions are in CELL UNITS relative to the grid origin (x_cell = x_m / cell_size);
 *     velocities in m/s.  Integral coordinates belong to the upper cell (A-4).
 *   - all floating-point state and outputs are IEEE binary32 (f32).
 *   - random draws: Philox4x32-10 keyed by the 64-bit seed, counter (index, k, stage, k>>32) (A-20),
 *     so the CPU oracle reproduces every draw bit for bit.
 *
 * Status codes: every function returns int, DOG_OK (0) on success, < 0 on error.  No C++ types or
 * exceptions cross this boundary.  A context is not thread-safe; distinct contexts are independent.
 */
#ifndef DOG_H
#define DOG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOG_OK        0
#define DOG_E_INVAL  (-1) /* invalid argument: sizes <= 0, C >= 2^31-1, probabilities out of range,
                             non-positive dt, NaN parameters, null pointers                        */
#define DOG_E_NOMEM  (-2) /* device or pinned-host allocation failed                             */
#define DOG_E_CUDA   (-3) /* a CUDA call failed; the context is poisoned (only dog_destroy)     */
#define DOG_E_NCCL   (-4) /* reserved: the library's own exchanges are peer-memory copies, not NCCL */
#define DOG_E_MEAS   (-5) /* a measurement cell was invalid (m_zO < 0, m_zF < 0, m_zO + m_zF >
                             1 + 2^-20, or NaN); such cells were treated as vacuous (0, 0).  Sticky
                             device flag, reported by the next synchronous call (dog_read_cells,
                             dog_get_state, dog_get_debug, dog_sync) and then cleared.           */
#define DOG_E_STATE  (-6) /* call-order misuse (e.g. sharded call on an unsharded context)      */

typedef struct dog_ctx dog_ctx;   /* opaque; created and owned by the library */

typedef struct {
    int32_t width, height;        /* cells; C = width*height, 1 <= C < 2^31-1 (see dog_create) */
    float   cell_size;            /* metres per cell, > 0 (Table I: 0.1 m)             */
    float   origin_x, origin_y;   /* world metres of the lower-left corner of cell (0, 0): the
                                     map between world and cell coordinates x = (X - origin_x) /
                                     cell_size; bookkeeping only (no kernel reads it), moved by
                                     dog_ego_scroll, read back with dog_get_origin               */
} dog_grid;

typedef struct {
    float p_s;             /* persistence probability in (0,1]         (Eq. 39; Table I 0.99)   */
    float p_b;             /* birth probability in [0,1)               (Eq. 67; 0.005..0.1)     */
    float sigma_pos;       /* m per (T/s); applied SD sigma_pos*T     (Table I 0.02; A-1)      */
    float sigma_vel;       /* (m/s) per (T/s); applied SD sigma_vel*T (Table I 0.8; A-1)       */
    float sigma_birth_vel; /* m/s, SD of new-born velocity            (Table I 4 m/s)          */
    float free_tau;        /* s, > 0: alpha(T) = exp(-T/free_tau); +INF gives alpha = 1 (A-9)  */
    float occ_max;         /* cap on predicted occupied mass, (0,1]; default 1 (Eq. 17; A-7)  */
    float v_max;           /* clamp of new-born |vx|,|vy| in m/s; <= 0 disables (A-16)         */
} dog_params;

/* dog_create -- allocate a filter in the empty initial state (A-19): all nu particles at the sentinel
 * position (-2^30 cells) with weight 0, m_F = 0, k = 0.
 *   grid, params : validated copies are kept (DOG_E_INVAL on violation; width, height <= 65535 (16-bit
 *                  rows / columns in the sort keys), width * height < 2^31 - 1 (u32 cell keys); the
 *                  masses' fixed point has 40 fractional bits below 2^24 cells and 63 - bitlen(C)
 *                  beyond, so every total stays below 2^64, A-23).
 *   n_particles  : nu, 1 <= nu < 2^30, persistent particles per cycle.
 *   n_birth      : nu_b, 0 <= nu_b < 2^30, new-born particles per cycle ("remains constant").
 *   seed         : Philox key (low 32 bits, high 32 bits).
 *   flags        : DOG_FLAG_DEBUG keeps per-stage device arrays for dog_get_debug (parity tests; whole-grid
 *                  contexts only); 0 for production (no extra traffic).
 *   n_devices, device_ids : 0 / NULL = one whole-grid context on the current device; 1 = on device_ids[0];
 *                  n >= 2 (<= 16, <= height) = a SHARDED context: the grid is cut into n row bands of
 *                  near-equal height (bottom-up), band s on device_ids[s] (ids may repeat: several bands on
 *                  one GPU).  Peer access is enabled between distinct devices (DOG_E_INVAL if the GPUs
 *                  cannot reach each other's memory).  Each band can hold all nu particles, so migration
 *                  cannot overflow and the owner-bucketed exchange reaches any band (no particle is lost).
 *                  A sharded context runs dog_step / dog_step_sharded / dog_read_cells(_sharded) /
 *                  dog_get_state / dog_set_state / dog_set_bands / dog_sync / dog_destroy; every other call
 *                  returns DOG_E_STATE.
 *   out          : receives the context; the context owns every device allocation it makes.
 * The caller's current device is unchanged on return. */
#define DOG_FLAG_DEBUG 1u
int dog_create(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
               uint64_t seed, uint32_t flags, int n_devices, const int* device_ids, dog_ctx** out);

/* dog_step_host_readout -- dog_step_host_async returning the FULL readout of each cycle (Alg. 3 / Alg. 6
 * stores): occ_host[C], free_host[C], mean_host[C][2], cov_host[C][3] (pinned HOST
 * buffers, any may be NULL), snapshot on the device and copied to the host on the copy stream while the
 * next cycle runs; complete after dog_sync(ctx, stream).  28 B per cell down, 8 B per cell up. */
int dog_step_host_readout(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, float* free_host,
                          float* mean_host, float* cov_host, void* stream);

/* ---- sharded contexts (multi-GPU) ----
 * dog_step_sharded -- one filter cycle on every band.  meas_band[s]: DEVICE pointer on device_ids[s] (or
 * peer-readable from it), float[rows of band s][width][2]; streams[s]: a cudaStream_t on device_ids[s].
 * Stream-ordered and asynchronous, with NO host synchronisation inside the cycle: the three couplings
 * of the bands (migrants after predict, born-mass totals for Alg. 5, joint-weight totals for Alg. 7)
 * move device to device over peer memory (NVLink), ordered by CUDA events between the streams.  The
 * union of the bands reproduces the whole-grid cycle bit for bit (Philox counters use global indices).
 * A failure mid-cycle poisons the context.
 * dog_step on a sharded context takes the whole-grid meas on device_ids[0] (read by every band over peer
 * memory) and a stream on device_ids[0]: the bands run on the context's own streams, forked from and
 * joined back into `stream`. */
int dog_step_sharded(dog_ctx* ctx, const float* const* meas_band, float dt, void* const* streams);
/* dog_read_cells_sharded -- each band's readouts into per-band DEVICE buffers on its device (any array
 * may be NULL; otherwise world entries, each possibly NULL).  Synchronises each band's stream.
 * dog_read_cells on a sharded context writes whole-grid buffers on device_ids[0] (peer copies). */
int dog_read_cells_sharded(dog_ctx* ctx, float* const* occ, float* const* free_mass, float* const* vel_mean,
                           float* const* vel_cov, void* const* streams);
/* dog_set_bands -- synchronous, between cycles (band rebalancing): move the band
 * boundaries to rows[0..world] (rows[0] = 0 < rows[1] < ... < rows[world] = height; any band height).
 * The state is carried over exactly (the global particle order does not change). */
int dog_set_bands(dog_ctx* ctx, const int32_t* rows);
/* dog_get_bands -- rows[world + 1] band bounds and (if devices != NULL) devices[world]; returns world
 * (1 for a whole-grid context). */
int dog_get_bands(dog_ctx* ctx, int32_t* rows, int* devices);
/* dog_world -- number of bands (1 for a whole-grid context). */
int dog_world(dog_ctx* ctx);

/* dog_step -- run one filter cycle.
 *   meas   : DEVICE pointer (same device as the context), float[height][width][2] =
 *            (m_zO, m_zF) per cell, row-major.  Read stream-ordered on `stream`; it must stay valid
 *            until the stream passes this step.  The library does not retain it.
 *   dt     : T in seconds, > 0 (A-29: all T-dependent scalars are recomputed per step).
 *   stream : cudaStream_t (0 = legacy default stream).  Asynchronous: returns after enqueueing. */
int dog_step(dog_ctx* ctx, const float* meas, float dt, void* stream);

/* dog_step_host -- the same cycle fed from HOST memory: copies meas (host, float[C][2]) to the
 * device, runs dog_step, and, if occ_host != NULL, copies the occupancy readout (float[C]) back;
 * synchronous on `stream`.  This is the end-to-end entry point (host buffers in, host result out). */
int dog_step_host(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, void* stream);

/* dog_step_host_async -- the pipelined end-to-end entry: the frame is copied host -> device on a copy
 * stream of the context (double-buffered staging) while the previous cycle runs on `stream`, and the
 * occupancy is snapshot on the device and copied device -> host on a second copy stream while the next
 * cycle runs.  Returns after enqueueing; meas_host must stay valid and unmodified, and occ_host is
 * complete, only after dog_sync(ctx, stream).  Use PINNED host buffers for overlap.  Whole-grid
 * contexts only. */
int dog_step_host_async(dog_ctx* ctx, const float* meas_host, float dt, float* occ_host, void* stream);

/* ---- row-band contexts: the band phases for callers that move the data themselves (one process per
 * GPU with a transport such as NCCL; paper_1605_02406_b200/shard.py).  A sharded context (above) drives
 * exactly these phases itself. ----
 * The grid is split into horizontal bands of rows, one context (and one GPU) per band.  A band context
 * owns its cells (m_F, readouts; the caller passes the band's measurement rows) and the particles whose
 * cell lies in the band.  The coupling between bands is exactly (i) particles that move into another
 * band during predict, (ii) the born-mass prefix of the bands below for the slot allocation
 * (Alg. 5, A-15) and (iii) the joint-weight prefix for systematic resampling (Alg. 7, A-24).  Philox
 * counters use global particle / slot indices, so the union of the bands reproduces the whole-grid
 * filter bit for bit.
 *   dog_band.row0/row1      : rows [row0, row1) of this band; rank/world: band index and count (bands
 *                             ordered bottom-up; rank 0 starts at row 0, the last ends at height).
 *   dog_band.lo_row0/hi_row1: first row of the band below / end row of the band above: migrants are
 *                             packed into four buckets -- to the band below, above, further below,
 *                             further above (owner-bucketed: no displacement is too large).
 *   dog_band.migrant_cap    : capacity, in particles, per bucket sent and per side received (< 2^26).
 * Call order per cycle: predict -> gather (the caller passes the neighbours' buckets, device pointers)
 * -> assign -> (caller all-gathers *mass_dev over the bands into mass_all[world], device) -> joint ->
 * (all-gather *weight_dev into weight_all[world]) -> resample.  Out-of-order calls return DOG_E_STATE.
 * Band contexts have no debug dumps (flags must be 0) and do not accept dog_step / dog_get_state
 * particle arrays; m_F and readouts work as usual on the band's cells.  A bucket or receive beyond
 * migrant_cap raises a device flag: the next dog_band_sizes / dog_sync / dog_read_cells returns
 * DOG_E_NOMEM and poisons the context (the cycle could not be completed exactly). */
typedef struct {
    int32_t row0, row1, rank, world, lo_row0, hi_row1;
    uint32_t migrant_cap;
} dog_band;
int dog_create_band(const dog_grid* grid, int64_t n_particles, int64_t n_birth, const dog_params* params,
                    uint64_t seed, uint32_t flags, const dog_band* band, dog_ctx** out);
/* phase 1: Alg. 1 for the own particles; migrants packed (device) into the four buckets. */
int dog_band_predict(dog_ctx* ctx, float dt, void* stream);
/* this band's four packed buckets (DEVICE float4 records (x, y, vx, vy) in global index order:
 * 0 below, 1 above, 2 further below, 3 further above) and their DEVICE u32 counts; valid once the
 * predict phase has run on its stream, until the next predict.  No synchronisation. */
int dog_band_outbox(dog_ctx* ctx, const float** rec, const uint32_t** cnt);
/* synchronises `stream` (after predict): the four bucket counts (host counts[4]) and the own particles of
 * this cycle -- for transports that must size their messages on the host. */
int dog_band_sizes(dog_ctx* ctx, uint32_t* counts, uint32_t* n_own, void* stream);
/* phase 1b (stream-ordered, no sync): assemble [from below | own | from above] from the other bands'
 * buckets -- DEVICE pointers readable from this band's device (its own memory, a peer GPU's, or a
 * transport's receive buffer) with DEVICE u32 counts:
 *   lo_near (+cnt): bucket 1 of band rank-1 (NULL for rank 0);  hi_near: bucket 0 of band rank+1 (NULL for
 *   the last band);  lo_far[n_lo_far = max(0, rank-1)]: bucket 3 of bands 0 .. rank-2 in band order;
 *   hi_far[n_hi_far = max(0, world-rank-2)]: bucket 2 of bands rank+2 .. world-1 in band order.
 * The far buckets are filtered to this band's rows (stable), so the local array stays in global index
 * order.  DOG_E_INVAL for a NULL / count mismatch. */
int dog_band_gather(dog_ctx* ctx, const float* lo_near, const uint32_t* lo_near_cnt, const float* hi_near,
                    const uint32_t* hi_near_cnt, int n_lo_far, const float* const* lo_far,
                    const uint32_t* const* lo_far_cnt, int n_hi_far, const float* const* hi_far,
                    const uint32_t* const* hi_far_cnt, void* stream);
/* phase 2: tile sort of [from below | own | from above], Alg. 3 on the band; *mass_dev = this band's
 * fixed-point born mass (device u64) to all-gather. */
int dog_band_assign(dog_ctx* ctx, const float* meas_band, const uint64_t** mass_dev, void* stream);
/* phase 2 of an exact PHD/MIB cycle (NEXT-3, dog_step_exact on a band): as dog_band_assign with the
 * band's rows of the observation grid obs_band[C_band][4] (DEVICE, 16-byte aligned) instead of the
 * measurement grid; the following joint and resample phases run the exact cycle's list handling. */
int dog_band_assign_exact(dog_ctx* ctx, const float* obs_band, const uint64_t** mass_dev, void* stream);
/* phase 2 of a Doppler cycle (NEXT-1, dog_step_doppler's branch on a band): as dog_band_assign, plus the
 * band's rows of the Doppler grid -- doppler_band[C_band][4] (16-byte aligned) and p_assoc_band[C_band],
 * DEVICE, valid until dog_band_resample has been enqueued; that phase then weights the band's Doppler
 * cells.  The joint weight of a band does not depend on the Doppler weights (A-35), so the exchanges
 * are those of the plain cycle. */
int dog_band_assign_doppler(dog_ctx* ctx, const float* meas_band, const float* doppler_band, const float* p_assoc_band,
                            const uint64_t** mass_dev, void* stream);
/* phase 3: slots on the global born-mass CDF, joint CDF of the band; *weight_dev = its joint weight. */
int dog_band_joint(dog_ctx* ctx, const uint64_t* mass_all_dev, const uint64_t** weight_dev, void* stream);
/* phase 4: moments, resampling of the band's share [F(P'), F(P' + W_band)) of the global outputs, births. */
int dog_band_resample(dog_ctx* ctx, const uint64_t* weight_all_dev, void* stream);
/* synchronous: own particles of the current state (float4 records, host) and the global index of the
 * first one; xyvv_host may be NULL to query the count. */
int dog_band_particles(dog_ctx* ctx, float* xyvv_host, uint64_t cap, uint32_t* n_own, uint64_t* global_first);
/* synchronous, between cycles (band rebalancing; resume): install a band's
 * state -- its own particles (n_own float4 records (x, y, vx, vy) from host, in global index order,
 * the first being global index global_first), m_free of its cells (host, C_band f32), the uniform
 * weight w_bar and the cycle counter k.  The particles must lie in the band's rows (the union of the
 * bands' states is the whole-grid state, cell-ordered).  DOG_E_INVAL for n_own beyond the band's
 * particle capacity or invalid values, DOG_E_STATE mid-cycle or on a whole-grid context.  The
 * readouts of the previous cycle are not moved (the next cycle rewrites them). */
int dog_band_set_state(dog_ctx* ctx, const float* xyvv_host, uint32_t n_own, uint64_t global_first,
                       const float* m_free_host, float w_bar, int64_t k);

/* ---- ego-motion compensation (SPEC ego_scroll) ----
 * dog_ego_scroll -- between cycles, move the grid content and the particles by the whole-cell part of
 * (dx, dy) + the stored residual (metres, grid axes; content moves by +shift): the integer part is fp64
 * truncation toward zero of (delta + residual) / cell_size, the fraction becomes the new residual
 * (A-32).  Cells scrolled in at the leading edge become vacuous (m_F = 0) with no particles;
 * particles leaving the grid become sentinel particles.  *shift_x / *shift_y (may be NULL) receive the
 * applied shift in cells.  DOG_E_INVAL (nothing changed) if a shift would reach half the grid side or
 * dx, dy are not finite.  Stream-ordered; whole-grid contexts only (DOG_E_STATE for a band).  The
 * readouts of the last cycle are not moved (they describe the cycle that produced them). */
int dog_ego_scroll(dog_ctx* ctx, double dx, double dy, int32_t* shift_x, int32_t* shift_y, void* stream);
int dog_ego_residual(dog_ctx* ctx, double* rx, double* ry);
/* dog_get_origin -- world metres of the lower-left corner of cell (0, 0) now: dog_grid's origin moved by
 * every applied ego shift (content moves by +shift cells, so the grid moves by -shift cell_size in the
 * world; fp64).  For band contexts the grid origin of the creating call (bands do not scroll). */
int dog_get_origin(dog_ctx* ctx, double* origin_x, double* origin_y);

/* ---- evaluation workload (PAPER section VIII, Eqs. 85-88) ----
 * dog_eval_cells -- per cell c of the context: the Mahalanobis distance m = v P^-1 v^T of the velocity
 * estimate (mean[c][2], cov[c][3] = var_x, var_y, cov_xy, Eqs. 81-84) from v = 0 (Eq. 88), computed in
 * fp64 and rounded to f32; P + 1e-6 I when det P <= 1e-12; m = 0 for a cell without moments (DESIGN.md
 * A-33).  mean_dev / cov_dev: DEVICE readouts (NULL: the filter's own, from its last cycle).  Which cells
 * have moments: valid_mode 1 = the filter's own record of its last cycle; valid_mode 0 = valid_dev[c] != 0
 * (u8, device), or if valid_dev is NULL, mean or cov nonzero.  Optional outputs: m_dev[C] (device f32);
 * with labels_dev[C] (u8: 0 unlabeled, 1 static, 2 dynamic) counts_host[n_thr][4] = (TP, FN, FP, TN) per
 * threshold thr_host[t] (dynamic detection: m >= thr; n_thr <= 64); with mask_dev[C] (u8: the cluster S)
 * sums_host[5] = (|S|, sum mean_x, sum var_x + mean_x^2, sum mean_y, sum var_y + mean_y^2) over cells of
 * S with moments (fp64, summation order unspecified), from which paper_1605_02406_b200/evaluate.py forms
 * Eqs. 85-87 and the ROC.  Synchronises `stream` when counts or sums are requested. */
int dog_eval_cells(dog_ctx* ctx, const float* mean_dev, const float* cov_dev, const uint8_t* valid_dev, int valid_mode,
                   const uint8_t* labels_dev, const uint8_t* mask_dev, const float* thr_host, int n_thr,
                   float* m_dev, uint64_t* counts_host, double* sums_host, void* stream);

/* dog_step_exact -- one cycle of the EXACT PHD/MIB filter (section V)
 * for a uniform single-object likelihood equal to the clutter density (the section IV-F setting,
 * P:795-867), on the same particle pipeline: the cell update is the Bernoulli update of Eqs. 31-32,
 * 38-42 instead of Dempster's rule (A-37), births are allocated wherever r_b > 0 (also in
 * unobserved cells), and m_F is not used.  obs: DEVICE f32 [C][4], 16-byte aligned, per cell
 * (occurred 0/1, p_TP, p_FP, unused) -- whether a measurement occurred in the cell and its true- /
 * false-positive probabilities, caller-guaranteed in [0, 1].  Readouts: occ = posterior
 * existence probability r (Eq. 42), free = 1 - r, moments as dog_step.  DOG_E_STATE for bands. */
int dog_step_exact(dog_ctx* ctx, const float* obs, float dt, void* stream);

/* dog_step_exact_lik -- one cycle of the exact PHD/MIB filter with a single-object likelihood (NEXT-3
 * general form; Eqs. 38, 49-52; A-38).  obs as dog_step_exact with
 * the 4th value the clutter density p_cl at the cell's measurement; plus two DEVICE arrays:
 *   lik[C][4] f32, 16-byte aligned: (u_x, u_y, v_r, sd) -- the measurement's radial-velocity likelihood
 *             g(z|x) = N(v.u - v_r; 0, sd^2) (Eq. 69), read only where p_assoc > 0 and occurred; finite,
 *             sd a normal positive f32 (as dog_step_doppler);
 *   p_assoc[C] f32: association probability p_A in [0, 1].
 * In a cell where a measurement occurred and p_A > 0: g_A(z|x) = p_A g(z|x) + (1 - p_A) p_cl, rho_p
 * and rho_b from the members' likelihood sum and the birth prior's expected likelihood (Eqs. 50-52),
 * the members' weights proportional to g_A (the Doppler Q_j split with the effective association
 * weight), and the associated births' radial velocity drawn from the posterior given z.  Every other
 * cell takes dog_step_exact's update; p_assoc all 0 gives exactly dog_step_exact.  Whole-grid contexts
 * only (DOG_E_STATE for bands); working buffers (20 B per particle slot + 28 B per cell) are allocated
 * on first use (DOG_E_NOMEM).  DOG_E_INVAL for a NULL or misaligned argument or an invalid dt. */
int dog_step_exact_lik(dog_ctx* ctx, const float* obs, const float* lik, const float* p_assoc, float dt,
                       void* stream);

/* dog_step_doppler -- one cycle with the Doppler / association branch (Eqs. 69-80,
 * P:1157-1232; A-34..A-36).  As dog_step, plus two DEVICE arrays:
 *   doppler[C][4] f32, 16-byte aligned: (u_x, u_y, v_r, sd) per cell -- unit radial direction, measured
 *                 radial speed (m/s) and its SD (a normal positive f32), read only where p_assoc > 0;
 *                 finite values required (results for NaN / infinite entries are unspecified);
 *   p_assoc[C]    f32: association probability p_A in [0, 1]; 0 = the cell has no Doppler measurement.
 * In a cell with p_A > 0 the persistent members are weighted by the Doppler likelihood g of their
 * predicted velocity (Eq. 71: w = p_A mu_A g w + (1 - p_A) mu_Abar w; A-35) and its birth slots split
 * into associated (velocity drawn around the measured radial speed) and unassociated ones (A-36).
 * p_assoc all 0 gives exactly dog_step's cycle.  Whole-grid contexts only (DOG_E_STATE for bands);
 * the working buffers (20 B per particle slot + 12 B per cell) are allocated on first use
 * (DOG_E_NOMEM).  DOG_E_INVAL for a NULL or misaligned argument or an invalid dt. */
int dog_step_doppler(dog_ctx* ctx, const float* meas, const float* doppler, const float* p_assoc, float dt,
                     void* stream);

/* dog_read_cells -- copy the readouts of the last completed cycle (posterior, before resampling,
 * P:1444) into caller DEVICE buffers (any may be NULL):
 *   occ[C] = m_O, free_mass[C] = m_F (Eq. 63); vel_mean[C][2] = (mean_vx, mean_vy) (Eq. 81);
 *   vel_cov[C][3] = (var_x, var_y, cov_xy) (Eqs. 83-84).  Cells without persistent particles or with
 *   rho_p <= 0 report mean = cov = 0.  Synchronises `stream`; returns DOG_E_MEAS if the sticky
 *   measurement flag was raised since the last report. */
int dog_read_cells(dog_ctx* ctx, float* occ, float* free_mass, float* vel_mean, float* vel_cov,
                   void* stream);

/* dog_sync -- synchronise the context's work on `stream` and report deferred errors. */
int dog_sync(dog_ctx* ctx, void* stream);

int dog_destroy(dog_ctx* ctx);
const char* dog_error_string(int status);

/* ---- state I/O (checkpoint/resume and parity injection; synchronous, HOST buffers) ----
 * The canonical state S_k is: nu particles (x, y in cell units; vx, vy in m/s) in canonical order,
 * ONE weight w_bar shared by all particles (Eq. 57 makes resampled weights equal), m_free[C], k.
 * Because draws are counter-based, set_state(get_state()) resumes bit-exactly. */
int dog_get_state(dog_ctx* ctx, float* x, float* y, float* vx, float* vy, float* w_bar,
                  float* m_free, int64_t* k);
int dog_set_state(dog_ctx* ctx, const float* x, const float* y, const float* vx, const float* vy,
                  float w_bar, const float* m_free, int64_t k);

/* ---- per-stage debug dumps of the last cycle (requires DOG_FLAG_DEBUG; synchronous) ----
 * `what` selects the array; host_dst receives `bytes` (must be >= the array size).  Returns the
 * number of bytes written (>= 0) or an error. */
enum {
    DOG_DBG_PRED_X = 1, DOG_DBG_PRED_Y, DOG_DBG_PRED_VX, DOG_DBG_PRED_VY, /* f32 [nu], input order */
    DOG_DBG_KEY,        /* u32 [nu] cell key, C = outside the grid                      */
    DOG_DBG_PERM,       /* u32 [nu] input index of each cell-sorted slot                */
    DOG_DBG_OFFSETS,    /* u32 [C+1] first sorted slot of each cell                      */
    DOG_DBG_RHO_P,      /* f32 [C]                                                       */
    DOG_DBG_RHO_B,      /* f32 [C]                                                       */
    DOG_DBG_RP,         /* u64 [C] fixed-point persistent mass floor(rho_p 2^40) (A-23)  */
    DOG_DBG_RB,         /* u64 [C] fixed-point born mass, 0 unless m_zO > 0 (A-13)       */
    DOG_DBG_NB,         /* u32 [C] birth slots per cell (A-15)                           */
    DOG_DBG_BIRTH_X, DOG_DBG_BIRTH_Y, DOG_DBG_BIRTH_VX, DOG_DBG_BIRTH_VY, /* f32 [nu_b]     */
    DOG_DBG_JOINT_IDX,  /* u32 [nu] joint index selected by each resampled particle      */
    DOG_DBG_SCALARS     /* u64 [8]: W, U, A, meas_bad_count, w_pred bits, w_bar bits, k, n_in */
};
int64_t dog_get_debug(dog_ctx* ctx, int what, void* host_dst, size_t bytes);

/* ---- stage profiling (bench evidence) ----
 * dog_profile_begin enables per-stage CUDA events (recorded on the step's stream, no host sync) for up
 * to max_steps subsequent dog_step calls; dog_profile_end synchronises and returns, per stage, the
 * summed device time in ms (stage_ms[DOG_MAX_STAGES]) and the number of profiled steps.
 * dog_profile_stage_name(i) names stage i ("predict", "sort0", ... "resample"). */
#define DOG_MAX_STAGES 16
int dog_profile_begin(dog_ctx* ctx, int max_steps);
int dog_profile_end(dog_ctx* ctx, float* stage_ms, int* n_stages, int* n_steps);
const char* dog_profile_stage_name(dog_ctx* ctx, int i);

/* ---- library introspection ---- */
int dog_version(void);                 /* ABI version, currently 1 */
int dog_launches_per_step(dog_ctx* ctx); /* kernels one dog_step launches (bench evidence) */

/* dog_check_transforms -- device self-check of the random-number transforms: the
 * kernels' range-specialised division and square root inside ln(m 2^-24) and the Box-Muller radius are
 * compared with IEEE div.rn / sqrt.rn for EVERY odd m in [1, 2^24) (the full input domain), and the
 * packed two-lane Box-Muller used by the predict kernel with two scalar evaluations over every odd m
 * and every sincos argument n in [0, 2^24).  Writes host bad[4] = (ln mismatches, sqrt mismatches,
 * packed mismatches, first failing index or ~0).  Runs on the current device, synchronously; no
 * context needed. */
int dog_check_transforms(uint64_t* bad_host);

#ifdef __cplusplus
}
#endif
#endif /* DOG_H */
