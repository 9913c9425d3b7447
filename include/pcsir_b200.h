/*
 * pcsir_b200.h — C ABI of the B200-native pcSIR / SIR filter step.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void* so this header needs no CUDA include). States are float32
 * structure-of-arrays: component c of particle i lives at states[c*ld + i]
 * with c in {0:x, 1:y, 2:vx, 3:vy, 4:I0} (state.py:16).
 *
 * Status codes: 0 ok, 1 invalid argument, 2 CUDA error, 3 out of memory,
 * 4 capacity exceeded (fused path: caller must use the general path).
 * pcs_last_error() returns a thread-local message for the last failure.
 *
 * Each function cites the reference interface it replaces
 * (paths relative to the reference repo, pkg/src/pcsir/).
 */
#ifndef PCSIR_B200_H
#define PCSIR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCS_OK 0
#define PCS_E_INVALID 1
#define PCS_E_CUDA 2
#define PCS_E_NOMEM 3
#define PCS_E_CAPACITY 4

/* device-side status flags (pcs_track_result_t.flags) */
#define PCS_FLAG_DEGENERATE 1u  /* all weights vanished  (filtering.py:70-71,82-83) */
#define PCS_FLAG_NONFINITE 2u   /* NaN state / likelihood (filtering.py:57-58)      */
#define PCS_FLAG_CAPACITY 4u    /* bin window / occupied bins exceeded fused capacity */
#define PCS_FLAG_RANGE 8u       /* |state| beyond the exact fixed-point range (2^24) */

typedef struct pcs_ctx pcs_ctx;

/* BinGrid (binning.py:28-77) */
typedef struct pcs_grid_t {
  double origin_x, origin_y, cell_width, cell_height;
  int64_t n_cols, n_rows;
} pcs_grid_t;

/* DynamicsParams (state.py:91-112) */
typedef struct pcs_dynamics_t {
  double sigma_pos, sigma_vel, sigma_int, dt;
} pcs_dynamics_t;

/* Likelihood models. model 0 = SpotLikelihood (imaging.py:111-140):
 * exp(-ssd/(2 sigma_xi^2)) over the clamped (2hw+1)^2 window.
 * model 1 = erf-integrated PSF, Poisson log-likelihood ratio (config 3, new).
 * model 2 = mid-point 4x4 sub-pixel PSF, Poisson (config 3 variant, new). */
typedef struct pcs_spot_t {
  double sigma_psf, i_bg, sigma_xi;
  int32_t halfwidth;
  int32_t model;         /* 0 gauss-ssd, 1 erf-poisson, 2 midpoint4x4-poisson;
                            | PCS_LIK_F64: Poisson models in float64 (the pcSIR
                            cell form; the fused pcSIR loop always uses it) */
} pcs_spot_t;
#define PCS_LIK_F64 16

/* InitSpec (state.py:140-161): mode 0 point, 1 uniform(width), 2 gauss(sigma) */
typedef struct pcs_init_t {
  double center[5];
  int32_t mode;
  int32_t pad_;
  double width, sigma;
} pcs_init_t;

/* ------------------------------------------------------------------ */
const char* pcs_last_error(void);
int pcs_version(void);
/* sizeof of the public structs, in this order: pcs_grid_t, pcs_dynamics_t,
 * pcs_spot_t, pcs_init_t, pcs_track_cfg_t, pcs_track_result_t (a binding
 * checks its layouts against them); returns how many were written. */
int pcs_abi_struct_sizes(int64_t* out, int32_t n);
int pcs_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor);

int pcs_ctx_create(pcs_ctx** out, int device);
int pcs_ctx_destroy(pcs_ctx* ctx);

/* ---- RNG (replay entry points; the same device functions feed the kernels) */
/* The normals pcs_propagate uses at (seed, frame) for particles
 * [index_offset, index_offset+n): out[c*ld + i], c = 0..4. Replaces the
 * rng.normal(size=(N,5)) draw at state.py:125. */
int pcs_philox_normals(uint64_t seed, uint32_t frame, int64_t index_offset, int64_t n,
                       float* out, int64_t ld, void* stream);
/* The two init normals (gauss) / uniforms (uniform) per particle
 * (state.py:171,173): out[c*ld + i], c = 0..1 (float32 normals) */
int pcs_philox_init_normals(uint64_t seed, int64_t index_offset, int64_t n, float* out,
                            int64_t ld, void* stream);
int pcs_philox_init_uniforms(uint64_t seed, int64_t index_offset, int64_t n, double* out,
                             int64_t ld, void* stream);
/* systematic offset u (filtering.py:99) and multinomial points (filtering.py:97) */
double pcs_philox_resample_u(uint64_t seed, uint32_t frame);
int pcs_philox_multinomial_points(uint64_t seed, uint32_t frame, int64_t n, double* out,
                                  void* stream);

/* ---- scene synthesis (synthesis.py:124-150: render_clean_frame +
 * render_sequence, generalised to several spots per frame). spots: device
 * float64 [n_frames][n_spots][3] = (x, y, I0); out: device float32
 * [n_frames][height][width]. Ideal frame = i_bg + sum of I0 gx gy over each
 * spot's +-ceil(window_sigmas * sigma_psf) window (exact order-free fixed-point
 * sum at 2^-32); noise != 0 draws Poisson(ideal) per pixel from the Philox
 * stream (seed, pixel, frame0 + k) plus optional Gaussian read noise clamped
 * at 0. */
int pcs_render_frames(pcs_ctx* ctx, const double* spots, int64_t n_spots, int64_t n_frames,
                      int64_t width, int64_t height, double sigma_psf, double i_bg,
                      double window_sigmas, int noise, double read_noise_std, uint64_t seed,
                      uint32_t frame0, float* out, void* stream);

/* ---- init_particle_set (state.py:164-175) */
int pcs_init_particles(const pcs_init_t* init, uint64_t seed, int64_t index_offset, int64_t n,
                       float* states, int64_t ld, void* stream);

/* ---- propagate_array (state.py:115-127) fused with the resampling gather
 * (filtering.py:107): out[:, j] = propagate(in[:, anc[j]]). anc may be NULL. */
int pcs_propagate(const float* states_in, float* states_out, int64_t ld, int64_t n,
                  const int32_t* ancestors, const pcs_dynamics_t* dyn, uint64_t seed,
                  uint32_t frame, int64_t index_offset, void* stream);

/* replay form of pcs_propagate: the five normals per particle are supplied
 * (normals[c*ldz + i]) instead of drawn — runs the device arithmetic on a
 * reference's recorded rng.normal draws (parity tests). */
int pcs_propagate_given(const float* states_in, float* states_out, int64_t ld, int64_t n,
                        const int32_t* ancestors, const pcs_dynamics_t* dyn,
                        const float* normals, int64_t ldz, void* stream);

/* ---- gather (filtering.py:107): out[:, j] = in[:, anc[j]] */
int pcs_gather(const float* states_in, float* states_out, int64_t ld, int64_t n,
               const int32_t* ancestors, void* stream);

/* ---- likelihood operator: kernels.spot_window_ssd (kernels.py:84-94,
 * _speedups.pyx:17-85). float64 in / float64 out, same window convention. */
int pcs_spot_window_ssd_f64(const double* pixels, int64_t height, int64_t width,
                            const double* xs, const double* ys, const double* i0s, int64_t n,
                            double sigma_psf, double i_bg, int32_t halfwidth, double* out,
                            void* stream);
/* float32 hot-path form: log-likelihood per state (SpotLikelihood.batch,
 * imaging.py:125-137, in the log domain). xs/ys/i0s are strided views
 * (e.g. rows of a SoA state block). */
int pcs_loglik(const float* pixels, int64_t height, int64_t width, const float* xs,
               const float* ys, const float* i0s, int64_t n, const pcs_spot_t* spot,
               double* out_loglik, void* stream);

/* ---- _partition + _dummy_states (binning.py:97-112,157-172), general
 * sort path (any grid size, 64-bit keys).
 * Outputs (capacity n each): flat[n] (u64 cell id per particle),
 * order[n] (stable argsort), bin_of[n] (occupied-bin rank of particle i),
 * unique[m], starts[m], counts[m]; *m_out = number of occupied bins.
 * Synchronises the stream to read m. */
int pcs_partition(pcs_ctx* ctx, const float* states, int64_t ld, int64_t n,
                  const pcs_grid_t* grid, uint64_t* flat, int32_t* order, int32_t* bin_of,
                  uint64_t* unique, int64_t* starts, int64_t* counts, int64_t* m_out,
                  void* stream);
/* dummies[c*ldd + b] (float32) for the m occupied bins. placement 0 = CoM,
 * 1 = cell centre. prior_w (float32, may be NULL) selects weighted CoM. */
/* Mid-point approximation bound study (bounds.py:116-180), built-in fields
 * in parametric form: kind 0 = a x^2 + b y^2 + c x + d y + e (params a..e),
 * 1 = sin(x) sin(y), 2 = i0 exp(-((x-x0)^2+(y-y0)^2)/(2 s2)) + i_bg (params
 * i0, i_bg, x0, y0, s2); params: host double[6].
 * pcs_bounds_deriv_max: max |f_xx|, max |f_yy| over np.linspace grids
 *   (derivative_maxima's sampling), out2: host double[2].
 * pcs_bounds_midpoint: signed mid-point error per cell (row-major n_rows x
 *   n_cols) by q x q Gauss-Legendre quadrature; edges / nodes / weights /
 *   cell_err are device float64 arrays. */
int pcs_bounds_deriv_max(int32_t kind, const double* params, double x_lo, double x_hi, int64_t nx,
                         double y_lo, double y_hi, int64_t ny, double* out2, void* stream);
int pcs_bounds_midpoint(int32_t kind, const double* params, const double* x_edges, int64_t n_cols,
                        const double* y_edges, int64_t n_rows, const double* nodes,
                        const double* weights, int32_t q, double* cell_err, void* stream);
/* make_dummy (binning.py:129-154): the representative state of ONE cell's
 * members. members: device float64 (n, 5) row-major; weights: device
 * float64 (n,) or NULL; placement 0 centre of mass, 1 cell centre (bounds =
 * host x_lo, x_hi, y_lo, y_hi); out: device float64 (5,). Reference
 * summation orders (np.add.reduceat rows, numpy pairwise weight total). */
int pcs_make_dummy(const double* members, int64_t n, const double* weights, int32_t placement,
                   const double* bounds, double* out, void* stream);
int pcs_dummies(pcs_ctx* ctx, const float* states, int64_t ld, int64_t n, const int32_t* order,
                const int32_t* bin_of, const int64_t* counts, const uint64_t* unique, int64_t m,
                const pcs_grid_t* grid, int32_t placement, const float* prior_w,
                float* dummies, int64_t ldd, void* stream);

/* ---- weights (filtering.py:62-90, binning.py:189-194) */
/* logw[i] = log(prior) + loglik[idx(i)] in float64, idx = bin_of (pcSIR
 * broadcast) or identity (bin_of NULL). The prior is prior_logw (float64
 * log-weights) if given, else prior_w (float32 linear weights) if given,
 * else uniform (constant dropped). */
int pcs_weight_update(const float* prior_w, const double* prior_logw, const double* loglik,
                      const int32_t* bin_of, int64_t n, double* logw, void* stream);
/* normalize (filtering.py:75-85) in the log domain; writes float32
 * normalised weights and returns max/normaliser. *degenerate set when every
 * weight is zero. Synchronises. */
int pcs_normalize(pcs_ctx* ctx, const double* logw, int64_t n, float* w_out, double* max_out,
                  double* norm_out, int32_t* degenerate, void* stream);
/* posterior_mean (filtering.py:112-114) and effective_sample_size
 * (filtering.py:88-90), exact fixed-point sums. Synchronises. */
int pcs_estimate_ess(pcs_ctx* ctx, const float* states, int64_t ld, const float* w, int64_t n,
                     double* est5_out, double* ess_out, void* stream);
/* _resample_indices (filtering.py:93-100): systematic with offset u, or
 * multinomial with Philox points (seed, frame). ancestors[n] int32. */
int pcs_resample_systematic(pcs_ctx* ctx, const float* w, int64_t n, double u,
                            int32_t* ancestors, void* stream);
int pcs_resample_multinomial(pcs_ctx* ctx, const float* w, int64_t n, const double* points,
                             int32_t* ancestors, void* stream);
/* materialise the exact cumulative weights (cdf[-1] forced to 1.0) */
int pcs_cdf(pcs_ctx* ctx, const float* w, int64_t n, double* cdf, void* stream);

/* ---- fused filter (sir_track filtering.py:176-182 / pcsir_track
 * binning.py:212-226; any ResampleConfig threshold, systematic or multinomial).
 * frames: K x H x W float32 device. Outputs (device): est[K*5] f64,
 * ess[K] f64, resampled[K] u8, occupied[K] i64 (likelihood evals per frame).
 * method 0 = SIR, 1 = pcSIR. Returns PCS_E_CAPACITY (with flags) when a
 * frame needs the general path. */
typedef struct pcs_track_cfg_t {
  int32_t method;        /* 0 SIR, 1 pcSIR */
  int32_t placement;     /* 0 CoM, 1 cell centre */
  int64_t n_particles;
  pcs_init_t init;
  pcs_dynamics_t dyn;
  pcs_spot_t spot;
  pcs_grid_t grid;
  uint64_t seed;
  uint32_t frame0;       /* frame counter offset for the RNG streams */
  int32_t use_graph;     /* capture one frame as a CUDA graph and replay it */
  double threshold_fraction;  /* resample when ESS < threshold_fraction * N
                                 (filtering.py:169-170); 0 means 1.0 */
  int32_t scheme;        /* 0 systematic, 1 multinomial (filtering.py:96-100) */
  int32_t weighted_com;  /* pcSIR: 1 = dummies at the prior-weighted centre of mass
                            (binning.py:160-165,186); fused while the prior weights
                            are uniform, PCS_E_CAPACITY (general path) otherwise */
} pcs_track_cfg_t;

typedef struct pcs_track_result_t {
  uint32_t flags;
  int32_t first_bad_frame;
  int64_t likelihood_evals;
} pcs_track_result_t;

int pcs_track(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, const float* frames, int64_t n_frames,
              int64_t height, int64_t width, double* est, double* ess, uint8_t* resampled,
              int64_t* occupied, pcs_track_result_t* result, void* stream);

/* Same as pcs_track but runs frames [k0, k1) only and keeps the filter
 * state inside ctx (pcs_track_begin initialises it). Used by the bench to
 * time individual steps. */
int pcs_track_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t height, int64_t width,
                    void* stream);
int pcs_track_steps(pcs_ctx* ctx, const float* frames, int64_t k0, int64_t k1, double* est,
                    double* ess, uint8_t* resampled, int64_t* occupied, void* stream);
int pcs_track_end(pcs_ctx* ctx, pcs_track_result_t* result, void* stream);
/* pcs_track_steps without graph replay, with a CUDA event around every
 * kernel: kernel_ms[i] accumulates the device time of launch i of the frame
 * (names from pcs_track_kernel_name). Synchronises after every frame. */
int pcs_track_steps_timed(pcs_ctx* ctx, const float* frames, int64_t k0, int64_t k1, double* est,
                          double* ess, uint8_t* resampled, int64_t* occupied, double* kernel_ms,
                          int32_t max_kernels, void* stream);
const char* pcs_track_kernel_name(pcs_ctx* ctx, int32_t i);
/* phase timestamps (globaltimer ns) recorded by the fused bins kernel */
int pcs_track_debug(pcs_ctx* ctx, int64_t* out16, void* stream);
/* launch geometry of the fused loop and which of its size-dependent code
 * paths ran (out[n], n >= 12): [0] step-1 CTAs, [1] step-1 warp tile
 * (particles), [2] step-1 warp tiles per warp (mean, rounded up), [3]
 * resampler CTAs, [4] resampler tiles per CTA (max; >= 2 runs the TMA ring
 * past its first buffer pair; 1 for the one-tile small form), [5] SIR
 * likelihood chunk (0: grid stride), [6] step-1 per-cell exchange flushes so
 * far (device), [7] most occupied cells of a frame so far (device), [8] cells
 * capacity of the fused loop, [9] step-1 per-cell flush period (members), [10]
 * SIR likelihood CTAs, [11] launches per frame. Synchronises the stream. */
int pcs_track_info(pcs_ctx* ctx, int64_t* out, int32_t n, void* stream);
/* kernel launches per fused step (for gpu_launches accounting) */
int pcs_track_launches_per_step(pcs_ctx* ctx);
/* export the current particle states / last ancestors of a running track */
int pcs_track_states(pcs_ctx* ctx, float** states, int64_t* ld);

/* ---- batched multi-target pcSIR (config 4, new; the reference tracks one
 * spot per filter). n_targets independent filters of
 * cfg->n_particles each, one CTA per target per frame. centers[t*5 + c] is
 * target t's InitSpec centre (mode/width/sigma from cfg->init). Target t's
 * RNG key is cfg->seed + (target_offset + t) * 0x9E3779B97F4A7C15, so it
 * equals pcs_track with that seed. Targets of different ranks are
 * independent (no communication). */
int pcs_mt_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t n_targets,
                 const double* centers, int64_t target_offset, int64_t n_frames, int64_t height,
                 int64_t width, void* stream);
int pcs_mt_step(pcs_ctx* ctx, const float* frame, int64_t k, void* stream);
int pcs_mt_results(pcs_ctx* ctx, double* est, double* ess, uint8_t* resampled, int64_t* occupied,
                   uint32_t* flags, int64_t* evals, void* stream);

/* ---- particle-sharded giant filter (config 5, new; pcs_shard.cuh) -------
 * Rank `rank` of `world` holds global particles [rank n, (rank+1) n)
 * (n = cfg->n_particles, n_global = world n). Per frame k, stream-ordered,
 * no host synchronisation, fixed-size collectives between the calls:
 *   pcs_shard_step1(frame k)      -> box: device int64[5]     (all-reduce MAX)
 *   pcs_shard_export(box)         -> limbs: device int64[wcap*16] (all-reduce SUM)
 *   pcs_shard_import_bins(box, limbs)   (identical bins stage on every rank)
 *   threshold_fraction < 1 only (frames whose particles carry prior weights,
 *   filtering.py:169-171; neutral values on the other frames):
 *     pcs_shard_prior(0)          -> out int64[1] max log-weight     (all-reduce MAX)
 *     pcs_shard_prior(1, in)      -> out int64[3] normaliser limbs   (all-reduce SUM)
 *     pcs_shard_prior(2, in)      -> out int64[18] estimate / ESS limbs (SUM),
 *                                    out_mm int64[2] weight range       (MAX)
 *     pcs_shard_prior(3, in, in_mm)  finalises the frame on every rank
 *   pcs_shard_total()             -> total: device int64[3]   (all-gather -> totals[world*3])
 *   systematic (scheme 0):
 *     pcs_shard_emit(totals)      -> send_prev / send_next: device float32[5*bcap+1]
 *                                    (send to rank-1 / rank+1, receive recv_prev
 *                                    from rank-1, recv_next from rank+1)
 *     pcs_shard_unpack(recv_prev, recv_next)
 *   multinomial (scheme 1; bcap = requests per rank pair):
 *     pcs_shard_route(totals)     -> req int32[world*(1+bcap)]        (all-to-all)
 *     pcs_shard_serve(req_in)     -> resp float32[world*5*bcap]      (all-to-all)
 *     pcs_shard_install(resp_in)
 * Results (est/ess/resampled/occupied rows) and flags as for pcs_track;
 * pcs_track_end reads the flags (all-reduce them so every rank raises). */
int pcs_shard_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t height, int64_t width,
                    int32_t rank, int32_t world, int64_t n_global, int64_t wcap, int64_t bcap,
                    void* stream);
int pcs_shard_step1(pcs_ctx* ctx, const float* frame, int64_t k, double* est, double* ess,
                    uint8_t* resampled, int64_t* occupied, int64_t* box, void* stream);
int pcs_shard_export(pcs_ctx* ctx, const int64_t* box, int64_t* limbs, void* stream);
int pcs_shard_import_bins(pcs_ctx* ctx, const int64_t* box, const int64_t* limbs, void* stream);
int pcs_shard_total(pcs_ctx* ctx, int64_t* total, void* stream);
int pcs_shard_emit(pcs_ctx* ctx, const int64_t* totals, float* send_prev, float* send_next,
                   void* stream);
int pcs_shard_unpack(pcs_ctx* ctx, const float* recv_prev, const float* recv_next, void* stream);
int pcs_shard_prior(pcs_ctx* ctx, int32_t stage, const int64_t* in, const int64_t* in_mm,
                    int64_t* out, int64_t* out_mm, void* stream);
int pcs_shard_route(pcs_ctx* ctx, const int64_t* totals, int32_t* req, void* stream);
int pcs_shard_serve(pcs_ctx* ctx, const int32_t* req_in, float* resp, void* stream);
int pcs_shard_install(pcs_ctx* ctx, const float* resp_in, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PCSIR_B200_H */
