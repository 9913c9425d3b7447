// pcs_capi.cu — extern "C" boundary of libpcsir_b200.so (see include/pcsir_b200.h).
//
// Host-side launch logic only; all arithmetic lives in the .cuh device code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>


#include "pcs_bin.cuh"
#include "pcs_synth.cuh"
#include "pcs_common.cuh"
#include "pcs_lik.cuh"
#include "pcs_state.cuh"
#include "pcs_multi.cuh"
#include "pcs_shard.cuh"
#include "pcs_sort.cuh"
#include "pcs_bounds.cuh"
#include "pcs_track.cuh"
#include "pcs_weights.cuh"

using namespace pcs;

static thread_local std::string g_last_error;
void pcs_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

#define PCS_CHECK_ARG(cond, msg)      \
  do {                                \
    if (!(cond)) {                    \
      pcs_set_last_error(msg);        \
      return PCS_E_INVALID;           \
    }                                 \
  } while (0)

#define PCS_LAUNCH_CHECK()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) {                                \
      pcs_set_last_error(cudaGetErrorString(_e));           \
      return PCS_E_CUDA;                                    \
    }                                                       \
  } while (0)

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

// ---------------------------------------------------------------------------
// context: device, SM count, grow-only scratch buffers, fused-track state
// ---------------------------------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct TrackState {
  bool active = false;
  pcs_track_cfg_t cfg{};
  TrackParams P{};
  BinsScratch bins{};
  int s1_grid = 0;
  int rs_grid = 0;       // k_sys_resample CTAs (all co-resident)
  int rs_small = 0;      // > 0: k_sys_resample_small with this many CTAs instead
  int red_grid = 0;      // k_sir_sum / k_sir_stats CTAs
  bool cond = false;     // pcSIR with threshold resampling (7-launch frame)
  int rs_grid2 = 0;      // k_sys_resample<2> CTAs in that mode
  static constexpr int MAX_LAUNCHES = 12;
  const char* names[MAX_LAUNCHES] = {};   // kernel of each launch of a frame
  int prop_grid = 0;
  int cells_grid = 0;    // k_pc_cells CTAs (8 warps each, one warp per occupied cell)
  bool s1_pow2 = false;  // k_pc_step1<true>: power-of-two cells, float32-exact origins
  int shard_rank = 0, shard_world = 1;   // sharded filter (pcs_shard_*)
  i64 shard_wcap = 0, shard_bcap = 0;
  double* shard_bnd = nullptr;     // multinomial: global cdf at the rank boundaries
  u32* shard_cnt = nullptr;        // multinomial: [world] requests, [world] sent
  int maxs = 0;
  i64 k = 0;             // host mirror of the frame counter
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  int launches = 0;
};

struct MtState {
  bool active = false;
  MtParams P{};
  int maxs = 0;
  i64 k = 0;
};

struct pcs_ctx {
  int device = 0;
  int sms = 148;
  std::vector<Buf> bufs;  // indexed scratch slots
  cudaStream_t cap = nullptr;
  TrackState tr;
  MtState mt;
  bool table_dirty = false;
  i64 table_cells = 0;
  u32* tab_cnt = nullptr;
  u64* tab_sum = nullptr;
  float* wtab = nullptr;
  u32* occ = nullptr;
};

enum Slot {
  SL_NORM = 0,
  SL_CUB,
  SL_SORT_KEYS,
  SL_SORT_IDX,
  SL_HEAD,
  SL_INCL,
  SL_NRUNS,
  SL_SUMS,
  SL_TILES,
  SL_PRE,
  SL_FLAGS,
  SL_TR_BUF0,
  SL_TR_BUF1,
  SL_TR_ANC,
  SL_TR_LL,
  SL_TR_PSLOT,
  SL_TR_CTL,
  SL_TR_TILES,
  SL_TR_PRE,
  SL_SHARD_ANC,
  SL_SHARD_BOX,
  SL_SHARD_BND,
  SL_SHARD_CNT,
  SL_MT_BUF0,
  SL_MT_BUF1,
  SL_MT_ANC,
  SL_MT_PSLOT,
  SL_MT_TGT,
  SL_MT_HASH,
  SL_MT_OUT,
  SL_MT_WPREV,
  SL_MT_LL,
  SL_MT_CDF,
  SL_SYNTH,
  SL_FMAP,
  SL_TR_WPREV,
  SL_TR_LLTAB,
  SL_TR_CDF,
  SL_TR_SUB,
  SL_SORT_KEYS2,
  SL_SORT_IDX2,
  SL_SCAN,
  SL_COUNT
};

static int scratch(pcs_ctx* c, int slot, size_t bytes, void** out) {
  if (c->bufs.size() < SL_COUNT) c->bufs.resize(SL_COUNT);
  Buf& b = c->bufs[slot];
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
      pcs_set_last_error(cudaGetErrorString(e));
      return PCS_E_NOMEM;
    }
    b.bytes = bytes;
  }
  *out = b.p;
  return PCS_OK;
}

#define PCS_SCRATCH(slot, bytes, ptr)                                   \
  do {                                                                  \
    void* _p = nullptr;                                                 \
    int _r = scratch(ctx, slot, (size_t)(bytes), &_p);                  \
    if (_r != PCS_OK) return _r;                                        \
    ptr = (decltype(ptr))_p;                                            \
  } while (0)

static inline int grid_for(i64 n, int block, int sms, int per_sm = 8) {
  i64 g = ceil_div(n, block);
  i64 cap = (i64)sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

static Grid to_grid(const pcs_grid_t* g) {
  Grid r;
  r.ox = g->origin_x;
  r.oy = g->origin_y;
  r.lx = g->cell_width;
  r.ly = g->cell_height;
  r.ncols = g->n_cols;
  r.nrows = g->n_rows;
  return r;
}

static Spot to_spot(const pcs_spot_t* s) {
  Spot r;
  r.sigma_psf = (float)s->sigma_psf;
  r.bg = (float)s->i_bg;
  r.inv2s2 = (float)(1.0 / (2.0 * s->sigma_psf * s->sigma_psf));
  r.inv_2sxi2 = 1.0 / (2.0 * s->sigma_xi * s->sigma_xi);
  r.hw = s->halfwidth;
  r.model = s->model & 15;
  r.f64 = (s->model & PCS_LIK_F64) ? 1 : 0;
  r.erf_scale = (float)(s->sigma_psf * 1.2533141373155002512078826);  // sigma*sqrt(pi/2)
  r.inv_sqrt2s = (float)(1.0 / (1.4142135623730950488 * s->sigma_psf));
  r.sigma64 = s->sigma_psf;
  r.bg64 = s->i_bg;
  r.inv2s2_64 = 1.0 / (2.0 * s->sigma_psf * s->sigma_psf);
  r.erf_scale64 = s->sigma_psf * 1.2533141373155002512078826;
  r.inv_sqrt2s64 = 1.0 / (1.4142135623730950488 * s->sigma_psf);
  return r;
}

static int maxs_for(int hw) {
  int S = 2 * hw + 1;
  if (S <= 9) return 9;
  if (S <= 11) return 11;
  if (S <= 15) return 15;
  return 0;
}

static int check_spot(const pcs_spot_t* s) {
  PCS_CHECK_ARG(s, "spot is NULL");
  PCS_CHECK_ARG(s->sigma_psf > 0, "sigma_psf must be > 0");
  PCS_CHECK_ARG(s->sigma_xi > 0, "sigma_xi must be > 0");
  PCS_CHECK_ARG(s->halfwidth >= 0, "halfwidth must be >= 0");
  const int m = s->model & ~PCS_LIK_F64;
  PCS_CHECK_ARG(m >= 0 && m <= 2, "unknown likelihood model");
  PCS_CHECK_ARG(m == 0 || s->i_bg > 0, "Poisson likelihood needs i_bg > 0");
  PCS_CHECK_ARG(s->i_bg >= 0, "i_bg must be >= 0");
  return PCS_OK;
}

static int check_grid(const pcs_grid_t* g) {
  PCS_CHECK_ARG(g, "grid is NULL");
  PCS_CHECK_ARG(g->cell_width > 0 && g->cell_height > 0, "cell dimensions must be > 0");
  PCS_CHECK_ARG(g->n_cols >= 1 && g->n_rows >= 1, "grid extent must be >= 1 cell per axis");
  PCS_CHECK_ARG((double)g->n_cols * (double)g->n_rows < 1.8e19, "grid has more than 2^64 cells");
  return PCS_OK;
}

extern "C" {

const char* pcs_last_error(void) { return g_last_error.c_str(); }
int pcs_version(void) { return 10000; }

int pcs_abi_struct_sizes(int64_t* out, int32_t n) {
  const int64_t sz[6] = {(int64_t)sizeof(pcs_grid_t),      (int64_t)sizeof(pcs_dynamics_t),
                         (int64_t)sizeof(pcs_spot_t),      (int64_t)sizeof(pcs_init_t),
                         (int64_t)sizeof(pcs_track_cfg_t), (int64_t)sizeof(pcs_track_result_t)};
  int k = 0;
  for (; out && k < n && k < 6; ++k) out[k] = sz[k];
  return k;
}

// ---- scene synthesis (synthesis.py:124-150) ----------------------------------
int pcs_render_frames(pcs_ctx* ctx, const double* spots, int64_t n_spots, int64_t n_frames,
                      int64_t width, int64_t height, double sigma_psf, double i_bg,
                      double window_sigmas, int noise, double read_noise_std, uint64_t seed,
                      uint32_t frame0, float* out, void* stream) {
  PCS_CHECK_ARG(ctx && out && n_frames >= 0 && n_spots >= 0 && width > 0 && height > 0,
                "bad arguments");
  PCS_CHECK_ARG(n_spots == 0 || spots, "spots is NULL");
  PCS_CHECK_ARG(sigma_psf > 0 && window_sigmas > 0 && read_noise_std >= 0, "bad psf parameters");
  cudaStream_t st = S(stream);
  const i64 npix = width * height;
  u64* acc = nullptr;
  PCS_SCRATCH(SL_SYNTH, npix * sizeof(u64), acc);
  const int r = (int)ceil(window_sigmas * sigma_psf);
  const double inv2s2 = 1.0 / (2.0 * sigma_psf * sigma_psf);
  const i64 work = n_spots * (i64)(2 * r + 1) * (2 * r + 1);
  for (i64 k = 0; k < n_frames; ++k) {
    PCS_CUDA_TRY(cudaMemsetAsync(acc, 0, npix * sizeof(u64), st));
    if (work > 0)
      k_synth_spots<<<grid_for(work, 256, ctx->sms), 256, 0, st>>>(spots + k * n_spots * 3, n_spots,
                                                                   width, height, inv2s2, r, acc);
    k_synth_finalize<<<grid_for(npix, 256, ctx->sms), 256, 0, st>>>(
        acc, npix, i_bg, noise, read_noise_std, seed, frame0 + (u32)k, out + k * npix);
  }
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor) {
  cudaDeviceProp p;
  PCS_CUDA_TRY(cudaGetDeviceProperties(&p, device));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return PCS_OK;
}

int pcs_ctx_create(pcs_ctx** out, int device) {
  PCS_CHECK_ARG(out, "out is NULL");
  PCS_CUDA_TRY(cudaSetDevice(device));
  pcs_ctx* c = new pcs_ctx();
  c->device = device;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) == cudaSuccess) c->sms = p.multiProcessorCount;
  c->bufs.resize(SL_COUNT);
  cudaError_t e = cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    pcs_set_last_error(cudaGetErrorString(e));
    return PCS_E_CUDA;
  }
  *out = c;
  return PCS_OK;
}

static void track_release(pcs_ctx* c) {
  if (c->tr.exec) cudaGraphExecDestroy(c->tr.exec);
  if (c->tr.graph) cudaGraphDestroy(c->tr.graph);
  c->tr.exec = nullptr;
  c->tr.graph = nullptr;
  c->tr.active = false;
}

int pcs_ctx_destroy(pcs_ctx* c) {
  if (!c) return PCS_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  track_release(c);
  for (auto& b : c->bufs)
    if (b.p) cudaFree(b.p);
  if (c->tab_cnt) cudaFree(c->tab_cnt);
  if (c->tab_sum) cudaFree(c->tab_sum);
  if (c->wtab) cudaFree(c->wtab);
  if (c->occ) cudaFree(c->occ);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// RNG replay
// ---------------------------------------------------------------------------
int pcs_philox_normals(uint64_t seed, uint32_t frame, int64_t off, int64_t n, float* out,
                       int64_t ld, void* stream) {
  PCS_CHECK_ARG(n >= 0 && out && ld >= n, "bad arguments");
  if (n == 0) return PCS_OK;
  k_philox_normals<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(seed, frame, off, n, out, ld);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_philox_init_normals(uint64_t seed, int64_t off, int64_t n, float* out, int64_t ld,
                            void* stream) {
  PCS_CHECK_ARG(n >= 0 && out && ld >= n, "bad arguments");
  if (n == 0) return PCS_OK;
  k_philox_init_normals<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(seed, off, n, out, ld);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_philox_init_uniforms(uint64_t seed, int64_t off, int64_t n, double* out, int64_t ld,
                             void* stream) {
  PCS_CHECK_ARG(n >= 0 && out && ld >= n, "bad arguments");
  if (n == 0) return PCS_OK;
  k_philox_init_uniforms<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(seed, off, n, out, ld);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

double pcs_philox_resample_u(uint64_t seed, uint32_t frame) {
  return philox_resample_u(seed, frame);
}

int pcs_philox_multinomial_points(uint64_t seed, uint32_t frame, int64_t n, double* out,
                                  void* stream) {
  PCS_CHECK_ARG(n >= 0 && out, "bad arguments");
  if (n == 0) return PCS_OK;
  k_philox_multinomial<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(seed, frame, n, out);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// init / propagate / gather
// ---------------------------------------------------------------------------
static InitSpecDev to_init(const pcs_init_t* init) {
  InitSpecDev d;
  for (int c = 0; c < 5; ++c) d.c[c] = init->center[c];
  d.mode = init->mode;
  d.width = init->width;
  d.sigma = init->sigma;
  return d;
}

int pcs_init_particles(const pcs_init_t* init, uint64_t seed, int64_t off, int64_t n,
                       float* states, int64_t ld, void* stream) {
  PCS_CHECK_ARG(init && states && n >= 1 && ld >= n, "bad arguments");
  PCS_CHECK_ARG(init->mode >= 0 && init->mode <= 2, "unknown init mode");
  PCS_CHECK_ARG(init->mode != 1 || init->width > 0, "uniform init needs width > 0");
  PCS_CHECK_ARG(init->mode != 2 || init->sigma > 0, "gauss init needs sigma > 0");
  k_init<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(to_init(init), seed, off, n, states, ld);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_propagate(const float* sin, float* sout, int64_t ld, int64_t n, const int32_t* anc,
                  const pcs_dynamics_t* dyn, uint64_t seed, uint32_t frame, int64_t off,
                  void* stream) {
  PCS_CHECK_ARG(sin && sout && dyn && n >= 1 && ld >= n, "bad arguments");
  PCS_CHECK_ARG(sin != sout, "in-place propagate is not supported");
  PCS_CHECK_ARG(dyn->sigma_pos >= 0 && dyn->sigma_vel >= 0 && dyn->sigma_int >= 0,
                "noise magnitudes must be >= 0");
  PCS_CHECK_ARG(dyn->dt > 0, "dt must be > 0");
  Dyn d = make_dyn(dyn->sigma_pos, dyn->sigma_vel, dyn->sigma_int, dyn->dt);
  int g = grid_for(n, 256, 148);
  if (anc)
    k_propagate<true><<<g, 256, 0, S(stream)>>>(sin, sout, ld, n, anc, d, philox_key(seed), frame, off);
  else
    k_propagate<false><<<g, 256, 0, S(stream)>>>(sin, sout, ld, n, nullptr, d, philox_key(seed), frame, off);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_propagate_given(const float* sin, float* sout, int64_t ld, int64_t n, const int32_t* anc,
                        const pcs_dynamics_t* dyn, const float* normals, int64_t ldz,
                        void* stream) {
  PCS_CHECK_ARG(sin && sout && dyn && normals && n >= 1 && ld >= n && ldz >= n, "bad arguments");
  PCS_CHECK_ARG(sin != sout, "in-place propagate is not supported");
  Dyn d = make_dyn(dyn->sigma_pos, dyn->sigma_vel, dyn->sigma_int, dyn->dt);
  k_propagate_given<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(sin, sout, ld, n, anc, d,
                                                                   normals, ldz);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_gather(const float* sin, float* sout, int64_t ld, int64_t n, const int32_t* anc,
               void* stream) {
  PCS_CHECK_ARG(sin && sout && anc && n >= 1 && ld >= n && sin != sout, "bad arguments");
  k_gather<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(sin, sout, ld, n, anc);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// likelihood
// ---------------------------------------------------------------------------
int pcs_spot_window_ssd_f64(const double* pixels, int64_t H, int64_t W, const double* xs,
                            const double* ys, const double* is, int64_t n, double sigma_psf,
                            double i_bg, int32_t hw, double* out, void* stream) {
  PCS_CHECK_ARG(pixels && xs && ys && is && out && H >= 1 && W >= 1 && n >= 0 && hw >= 0,
                "bad arguments");
  PCS_CHECK_ARG(sigma_psf > 0, "sigma_psf must be > 0");
  if (n == 0) return PCS_OK;
  double inv = 1.0 / (2.0 * sigma_psf * sigma_psf);
  k_ssd_f64<<<grid_for(n, 128, 148, 16), 128, 0, S(stream)>>>(pixels, H, W, xs, ys, is, n, inv,
                                                               i_bg, hw, out);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_loglik(const float* pixels, int64_t H, int64_t W, const float* xs, const float* ys,
               const float* is, int64_t n, const pcs_spot_t* spot, double* out, void* stream) {
  int r = check_spot(spot);
  if (r) return r;
  PCS_CHECK_ARG(pixels && xs && ys && is && out && H >= 1 && W >= 1 && n >= 0, "bad arguments");
  if (n == 0) return PCS_OK;
  Spot sp = to_spot(spot);
  int g = grid_for(n, 256, 148, 16);
  switch (maxs_for(spot->halfwidth)) {
    case 9: k_loglik<9><<<g, 256, 0, S(stream)>>>(pixels, H, W, xs, ys, is, n, sp, out); break;
    case 11: k_loglik<11><<<g, 256, 0, S(stream)>>>(pixels, H, W, xs, ys, is, n, sp, out); break;
    case 15: k_loglik<15><<<g, 256, 0, S(stream)>>>(pixels, H, W, xs, ys, is, n, sp, out); break;
    default: k_loglik<0><<<g, 256, 0, S(stream)>>>(pixels, H, W, xs, ys, is, n, sp, out);
  }
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// partition / dummies (general sort path)
// ---------------------------------------------------------------------------
// exclusive scan of n int32 in place: block partials, then the block totals
// scanned recursively (tmp holds every level's totals) and added back
static int scan_excl_i32(int* a, i64 n, int* tmp, cudaStream_t st) {
  const i64 nb = ceil_div(n, (i64)SC_BLOCK);
  k_scan_blocks<<<(unsigned)nb, SC_THREADS, 0, st>>>(a, n, tmp);
  PCS_LAUNCH_CHECK();
  if (nb > 1) {
    int r = scan_excl_i32(tmp, nb, tmp + nb, st);
    if (r) return r;
    k_scan_add<<<(unsigned)std::min<i64>(ceil_div(n, (i64)256), 65535), 256, 0, st>>>(a, n, tmp);
    PCS_LAUNCH_CHECK();
  }
  return PCS_OK;
}

int pcs_partition(pcs_ctx* ctx, const float* states, int64_t ld, int64_t n,
                  const pcs_grid_t* grid, uint64_t* flat, int32_t* order, int32_t* bin_of,
                  uint64_t* unique, int64_t* starts, int64_t* counts, int64_t* m_out,
                  void* stream) {
  int r = check_grid(grid);
  if (r) return r;
  PCS_CHECK_ARG(ctx && states && flat && order && bin_of && unique && starts && counts && m_out,
                "bad arguments");
  PCS_CHECK_ARG(n >= 1 && n < INT_MAX && ld >= n, "n out of range");
  cudaStream_t st = S(stream);
  Grid g = to_grid(grid);
  // hand-written stable LSD radix sort (pcs_sort.cuh) of (flat id, index)
  // pairs over the bits of the largest flat id, then the run partition
  u64 *ka, *kb;
  int *va, *vb, *incl, *scan_tmp;
  u32* flags;
  const i64 ntiles = ceil_div(n, (i64)RS8_TILE);
  PCS_SCRATCH(SL_SORT_KEYS, n * sizeof(u64), ka);
  PCS_SCRATCH(SL_SORT_KEYS2, n * sizeof(u64), kb);
  PCS_SCRATCH(SL_SORT_IDX, n * sizeof(int), va);
  PCS_SCRATCH(SL_SORT_IDX2, n * sizeof(int), vb);
  PCS_SCRATCH(SL_INCL, std::max<i64>(n, 256 * ntiles) * sizeof(int), incl);
  PCS_SCRATCH(SL_SCAN, (ceil_div(std::max<i64>(n, 256 * ntiles), (i64)SC_BLOCK - 1) + 64) * sizeof(int),
              scan_tmp);
  PCS_SCRATCH(SL_FLAGS, 64, flags);
  PCS_CUDA_TRY(cudaMemsetAsync(flags, 0, 4, st));
  const int gr = grid_for(n, 256, ctx->sms);
  k_cell_keys<<<gr, 256, 0, st>>>(states, ld, n, g, ka, va, flags);
  PCS_LAUNCH_CHECK();
  const u64 maxkey = (u64)grid->n_cols * (u64)grid->n_rows - 1ull;
  const int end_bit = maxkey ? 64 - clz64(maxkey) : 1;
  const int passes = (end_bit + 7) / 8;
  for (int ps = 0; ps < passes; ++ps) {
    k_radix_hist<<<(unsigned)ntiles, RS8_THREADS, 0, st>>>(ka, n, 8 * ps, ntiles, incl);
    PCS_LAUNCH_CHECK();
    int r = scan_excl_i32(incl, 256 * ntiles, scan_tmp, st);
    if (r) return r;
    // the last pass writes the caller's order array directly
    u64* kd = (ps == passes - 1) ? (u64*)flat : kb;
    int* vd = (ps == passes - 1) ? (int*)order : vb;
    k_radix_scatter<<<(unsigned)ntiles, RS8_THREADS, 0, st>>>(ka, va, kd, vd, n, 8 * ps, ntiles,
                                                              incl);
    PCS_LAUNCH_CHECK();
    if (ps < passes - 1) {
      std::swap(ka, kb);
      std::swap(va, vb);
    }
  }
  // flat (the caller's array) now holds the sorted keys: rebuild the
  // per-particle flat ids afterwards (binning.py:105 returns them unsorted)
  const u64* sorted = (const u64*)flat;
  u64* sorted_keep = kb;   // copy of the sorted keys (flat is overwritten below)
  PCS_CUDA_TRY(cudaMemcpyAsync(sorted_keep, sorted, n * sizeof(u64), cudaMemcpyDeviceToDevice, st));
  k_key_heads<<<gr, 256, 0, st>>>(sorted_keep, n, incl);
  PCS_LAUNCH_CHECK();
  int r2 = scan_excl_i32(incl, n, scan_tmp, st);
  if (r2) return r2;
  k_runs<<<gr, 256, 0, st>>>(sorted_keep, order, n, incl, (u64*)unique, (i64*)starts, bin_of);
  PCS_LAUNCH_CHECK();
  k_cell_keys<<<gr, 256, 0, st>>>(states, ld, n, g, (u64*)flat, va, flags);   // unsorted ids
  PCS_LAUNCH_CHECK();
  int last_rank = 0;
  u64 last2[2] = {0, 0};
  PCS_CUDA_TRY(cudaMemcpyAsync(&last_rank, incl + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaMemcpyAsync(last2, sorted_keep + (n >= 2 ? n - 2 : 0), (n >= 2 ? 2 : 1) * sizeof(u64),
                               cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  const bool last_head = (n == 1) || (last2[1] != last2[0]);
  const i64 m = (i64)last_rank + (last_head ? 1 : 0);
  k_run_counts<<<grid_for(m, 256, ctx->sms), 256, 0, st>>>((const i64*)starts, m, n, (i64*)counts);
  PCS_LAUNCH_CHECK();
  u32 hflags = 0;
  PCS_CUDA_TRY(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  *m_out = m;
  if (hflags & PCS_FLAG_NONFINITE) {
    pcs_set_last_error("non-finite particle position");
    return PCS_E_INVALID;
  }
  return PCS_OK;
}


int pcs_dummies(pcs_ctx* ctx, const float* states, int64_t ld, int64_t n, const int32_t* order,
                const int32_t* bin_of, const int64_t* counts, const uint64_t* unique, int64_t m,
                const pcs_grid_t* grid, int32_t placement, const float* prior_w, float* dummies,
                int64_t ldd, void* stream) {
  int r = check_grid(grid);
  if (r) return r;
  PCS_CHECK_ARG(ctx && states && order && bin_of && counts && unique && dummies, "bad arguments");
  PCS_CHECK_ARG(n >= 1 && m >= 1 && m <= n && ldd >= m && ld >= n, "bad sizes");
  PCS_CHECK_ARG(placement == 0 || placement == 1, "unknown placement");
  cudaStream_t st = S(stream);
  u64* sums;
  size_t sb = (size_t)6 * m * 2 * sizeof(u64);
  PCS_SCRATCH(SL_SUMS, sb, sums);
  PCS_CUDA_TRY(cudaMemsetAsync(sums, 0, sb, st));
  k_bin_sums<<<grid_for(n, 256, ctx->sms), 256, 0, st>>>(states, ld, n, order, bin_of, prior_w,
                                                          sums, m);
  PCS_LAUNCH_CHECK();
  k_dummies<<<grid_for(m, 256, ctx->sms), 256, 0, st>>>(sums, (const i64*)counts, (const u64*)unique, m, to_grid(grid),
                                                         placement, prior_w ? 1 : 0, dummies, ldd);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

static int to_field(int32_t kind, const double* params, FieldDev* F) {
  PCS_CHECK_ARG(params && kind >= 0 && kind <= 2, "field kind must be 0 (polynomial), 1 (sinsin) or 2 (gaussian)");
  F->kind = kind;
  for (int i = 0; i < 6; ++i) F->p[i] = params[i];
  if (kind == 2) PCS_CHECK_ARG(params[4] > 0.0, "gaussian field needs sigma^2 > 0");
  return PCS_OK;
}

int pcs_bounds_deriv_max(int32_t kind, const double* params, double x_lo, double x_hi, int64_t nx,
                         double y_lo, double y_hi, int64_t ny, double* out2, void* stream) {
  FieldDev F;
  int r = to_field(kind, params, &F);
  if (r) return r;
  PCS_CHECK_ARG(out2 && nx >= 1 && ny >= 1, "bad arguments");
  unsigned long long* d;
  cudaStream_t st = S(stream);
  PCS_CUDA_TRY(cudaMallocAsync((void**)&d, 16, st));
  PCS_CUDA_TRY(cudaMemsetAsync(d, 0, 16, st));
  k_deriv_max<<<grid_for(nx * ny, 256, 148, 8), 256, 0, st>>>(F, x_lo, x_hi, nx, y_lo, y_hi, ny, d);
  PCS_LAUNCH_CHECK();
  unsigned long long h[2];
  PCS_CUDA_TRY(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaFreeAsync(d, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(out2, h, 16);
  return PCS_OK;
}

int pcs_bounds_midpoint(int32_t kind, const double* params, const double* x_edges, int64_t n_cols,
                        const double* y_edges, int64_t n_rows, const double* nodes,
                        const double* weights, int32_t q, double* cell_err, void* stream) {
  FieldDev F;
  int r = to_field(kind, params, &F);
  if (r) return r;
  PCS_CHECK_ARG(x_edges && y_edges && nodes && weights && cell_err && n_cols >= 1 && n_rows >= 1 &&
                q >= 1, "bad arguments");
  const i64 cells = n_cols * n_rows;
  k_midpoint_error<<<(unsigned)std::min<i64>(ceil_div(cells, (i64)8), 148 * 64), 256, 0, S(stream)>>>(
      F, x_edges, n_cols, y_edges, n_rows, nodes, weights, q, cell_err);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_make_dummy(const double* members, int64_t n, const double* weights, int32_t placement,
                   const double* bounds, double* out, void* stream) {
  PCS_CHECK_ARG(members && out && bounds, "bad arguments");
  PCS_CHECK_ARG(n >= 1, "a dummy needs at least one member state");
  PCS_CHECK_ARG(placement == 0 || placement == 1, "unknown placement");
  k_make_dummy<<<1, 32, 0, S(stream)>>>(members, n, weights, placement, bounds[0], bounds[1],
                                        bounds[2], bounds[3], out);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// weights
// ---------------------------------------------------------------------------
int pcs_weight_update(const float* prior_w, const double* prior_logw, const double* ll,
                      const int32_t* bin_of, int64_t n, double* logw, void* stream) {
  PCS_CHECK_ARG(ll && logw && n >= 1, "bad arguments");
  k_weight_update<<<grid_for(n, 256, 148), 256, 0, S(stream)>>>(prior_w, prior_logw, ll, bin_of, n,
                                                                 logw);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_normalize(pcs_ctx* ctx, const double* logw, int64_t n, float* w, double* max_out,
                  double* norm_out, int32_t* degenerate, void* stream) {
  PCS_CHECK_ARG(ctx && logw && w && n >= 1, "bad arguments");
  cudaStream_t st = S(stream);
  NormCtl* nc;
  PCS_SCRATCH(SL_NORM, sizeof(NormCtl), nc);
  NormCtl h;
  memset(&h, 0, sizeof(h));
  h.max_ord = (i64)0x8000000000000000ll;  // below every encoded double
  PCS_CUDA_TRY(cudaMemcpyAsync(nc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  int g = grid_for(n, 256, ctx->sms);
  k_logw_max<256><<<g, 256, 0, st>>>(logw, n, nc);
  PCS_LAUNCH_CHECK();
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, nc, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  if (h.nonfinite) {
    pcs_set_last_error("likelihood values must be finite and >= 0");
    return PCS_E_INVALID;
  }
  double m = *(double*)&h.max_ord;
  {
    i64 i = h.max_ord;
    i64 raw = (i >= 0) ? i : (i ^ 0x7FFFFFFFFFFFFFFFll);
    memcpy(&m, &raw, 8);
  }
  if (!(m > -INFINITY)) {
    if (degenerate) *degenerate = 1;
    if (max_out) *max_out = m;
    if (norm_out) *norm_out = 0.0;
    return PCS_OK;
  }
  k_logw_sum<256><<<g, 256, 0, st>>>(logw, n, nc);
  PCS_LAUNCH_CHECK();
  k_logw_normalise<<<g, 256, 0, st>>>(logw, n, nc, w);
  PCS_LAUNCH_CHECK();
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, nc, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  if (degenerate) *degenerate = 0;
  if (max_out) *max_out = m;
  if (norm_out) {
    i128 Sv = (i128)(((u128)h.S[1] << 64) | (u128)h.S[0]);
    *norm_out = ldexp(i128_to_f64_rn(Sv), -FX_S);
  }
  return PCS_OK;
}

int pcs_estimate_ess(pcs_ctx* ctx, const float* states, int64_t ld, const float* w, int64_t n,
                     double* est5, double* ess, void* stream) {
  PCS_CHECK_ARG(ctx && states && w && n >= 1 && ld >= n, "bad arguments");
  cudaStream_t st = S(stream);
  NormCtl* nc;
  PCS_SCRATCH(SL_NORM, sizeof(NormCtl), nc);
  PCS_CUDA_TRY(cudaMemsetAsync(nc, 0, sizeof(NormCtl), st));
  k_estimate_ess<256><<<grid_for(n, 256, ctx->sms), 256, 0, st>>>(states, ld, w, n, nc);
  PCS_LAUNCH_CHECK();
  NormCtl h;
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, nc, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  for (int c = 0; c < 5; ++c) {
    i128 v = (i128)(((u128)h.est[c][1] << 64) | (u128)h.est[c][0]);
    if (est5) est5[c] = ldexp(i128_to_f64_rn(v), -(FX_WQ + FX_STATE));
  }
  i128 v2 = (i128)(((u128)h.w2[1] << 64) | (u128)h.w2[0]);
  if (ess) *ess = 1.0 / ldexp(i128_to_f64_rn(v2), -FX_W2);
  return PCS_OK;
}

static int cdf_pass(pcs_ctx* ctx, const float* w, int64_t n, double u, int32_t* anc, double* cdf,
                    int mode, cudaStream_t st) {
  i64 nt = ceil_div(n, SCAN_TILE);
  u128* tot;
  u128* pre;
  PCS_SCRATCH(SL_TILES, nt * sizeof(u128), tot);
  PCS_SCRATCH(SL_PRE, nt * sizeof(u128), pre);
  WeightSrc src;
  memset(&src, 0, sizeof(src));
  src.w = w;
  src.kind = 0;
  k_cdf_tiles<<<(unsigned)nt, SCAN_BLOCK, 0, st>>>(src, n, tot);
  PCS_LAUNCH_CHECK();
  k_scan_tiles<<<1, 1024, 0, st>>>(tot, nt, pre, nullptr);
  PCS_LAUNCH_CHECK();
  if (mode == 0)
    k_cdf_emit<0><<<(unsigned)nt, SCAN_BLOCK, 0, st>>>(src, n, pre, u, anc, nullptr);
  else
    k_cdf_emit<1><<<(unsigned)nt, SCAN_BLOCK, 0, st>>>(src, n, pre, u, nullptr, cdf);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_resample_systematic(pcs_ctx* ctx, const float* w, int64_t n, double u, int32_t* anc,
                            void* stream) {
  PCS_CHECK_ARG(ctx && w && anc && n >= 1 && n < INT_MAX, "bad arguments");
  PCS_CHECK_ARG(u >= 0.0 && u < 1.0, "u must be in [0, 1)");
  return cdf_pass(ctx, w, n, u, anc, nullptr, 0, S(stream));
}

int pcs_cdf(pcs_ctx* ctx, const float* w, int64_t n, double* cdf, void* stream) {
  PCS_CHECK_ARG(ctx && w && cdf && n >= 1, "bad arguments");
  return cdf_pass(ctx, w, n, 0.0, nullptr, cdf, 1, S(stream));
}

int pcs_resample_multinomial(pcs_ctx* ctx, const float* w, int64_t n, const double* points,
                             int32_t* anc, void* stream) {
  PCS_CHECK_ARG(ctx && w && points && anc && n >= 1 && n < INT_MAX, "bad arguments");
  cudaStream_t st = S(stream);
  double* cdf;
  PCS_SCRATCH(SL_SORT_KEYS, n * sizeof(double), cdf);
  int r = cdf_pass(ctx, w, n, 0.0, nullptr, cdf, 1, st);
  if (r) return r;
  k_searchsorted<<<grid_for(n, 256, ctx->sms), 256, 0, st>>>(cdf, n, points, anc);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}


// ---------------------------------------------------------------------------
// fused track (device-resident loop, one CUDA graph per frame)
// ---------------------------------------------------------------------------
__global__ void k_iota(int* a, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

__global__ void k_iota_mod(int* a, i64 n, i64 m) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    a[i] = (int)(i % m);
}

__global__ void k_ctl_init(TrackCtl* C, double cx, double cy) {
  memset(C, 0, sizeof(TrackCtl));
  reset_frame(C);
  C->first_bad = INT_MAX;
  C->center[0] = cx;
  C->center[1] = cy;
}

__global__ void k_ctl_io(TrackCtl* C, const float* frames, i64 kf, i64 ko, i64 kend, double* est,
                         double* ess, unsigned char* res, i64* occ, int fmap_ok = 0) {
  C->k_end = kend;
  C->fmap_ok = fmap_ok;
  C->frames = frames;
  C->k_frames = kf;
  C->k_out = ko;
  C->out_est = est;
  C->out_ess = ess;
  C->out_res = res;
  C->out_occ = occ;
}

// launch with the programmatic-stream-serialization attribute (PDL): the
// kernel may be scheduled before its predecessor in the stream has drained;
// it calls griddepcontrol.wait before consuming the predecessor's results
extern "C++" {
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // extern "C++"


// Enqueue one frame. If evs is non-null, evs[i] is recorded before launch i
// and evs[launches] after the last one (per-kernel CUDA-event timing).
// first: the track's first frame (step 1 queues the particles outside its sub-window)
static int enqueue_frame(pcs_ctx* ctx, cudaStream_t st, cudaEvent_t* evs = nullptr,
                         bool first = false) {
  TrackState& T = ctx->tr;
  TrackParams& P = T.P;
  int q = 0;
  auto mark = [&](const char* name) {   // event before launch q; its name for the timings
    if (evs) cudaEventRecord(evs[q], st);
    if (q < TrackState::MAX_LAUNCHES) T.names[q] = name;
    ++q;
  };
  if (T.cfg.method == 1) {
    mark("k_pc_step1");
    if (first) {
      if (T.s1_pow2) k_pc_step1<true, true><<<T.s1_grid, S1_THREADS, S1_SMEM_Q, st>>>(P);
      else k_pc_step1<false, true><<<T.s1_grid, S1_THREADS, S1_SMEM_Q, st>>>(P);
    } else {
      if (T.s1_pow2) k_pc_step1<true><<<T.s1_grid, S1_THREADS, S1_SMEM, st>>>(P);
      else k_pc_step1<false><<<T.s1_grid, S1_THREADS, S1_SMEM, st>>>(P);
    }
    mark("k_pc_cells");
    launch_pdl(k_pc_cells, T.cells_grid, CELLS_BLOCK, 0, st, P, T.bins);
    mark("k_pc_bins");
    launch_pdl(k_pc_bins, 1, BINS_BLOCK, 0, st, P, T.bins);
    if (T.cond) {
      // frames whose particles carry prior weights finish per particle (the
      // kernels of the other mode return at once)
      mark("k_pc_prior_ll");
      k_pc_prior_ll<<<T.red_grid, 256, 0, st>>>(P);
      mark("k_sir_sum");
      k_sir_sum<<<T.red_grid, 256, 0, st>>>(P);
      mark("k_sir_stats");
      k_sir_stats<<<T.red_grid, 256, 0, st>>>(P);
    }
    mark("k_sys_resample");
    if (T.rs_small) launch_pdl(k_sys_resample_small<1>, T.rs_small, SCAN_BLOCK, 0, st, P);
    else if (P.multinomial) launch_pdl(k_sys_resample<1, true>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<1>), st, P);
    else launch_pdl(k_sys_resample<1>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<1>), st, P);
    if (T.cond) {
      mark("k_sys_resample:prior");
      if (T.rs_small) launch_pdl(k_sys_resample_small<2>, T.rs_small, SCAN_BLOCK, 0, st, P);
      else if (P.multinomial) launch_pdl(k_sys_resample<2, true>, T.rs_grid2, SCAN_BLOCK, sizeof(RsSmem<2>), st, P);
      else launch_pdl(k_sys_resample<2>, T.rs_grid2, SCAN_BLOCK, sizeof(RsSmem<2>), st, P);
    }
    if (P.multinomial) {
      mark("k_multinomial_emit");
      k_multinomial_emit<<<grid_for(P.n, 256, ctx->sms), 256, 0, st>>>(P);
    }
  } else {
    mark("k_sir_propagate_lik");
    switch (T.maxs) {
      case 9: k_sir_propagate_lik<9><<<T.prop_grid, 256, 0, st>>>(P); break;
      case 11: k_sir_propagate_lik<11><<<T.prop_grid, 256, 0, st>>>(P); break;
      case 15: k_sir_propagate_lik<15><<<T.prop_grid, 256, 0, st>>>(P); break;
      default: k_sir_propagate_lik<0><<<T.prop_grid, 256, 0, st>>>(P);
    }
    mark("k_sir_sum");
    k_sir_sum<<<T.red_grid, 256, 0, st>>>(P);
    mark("k_sir_stats");
    k_sir_stats<<<T.red_grid, 256, 0, st>>>(P);   // its last CTA finalises the frame
    mark("k_sys_resample");
    if (T.rs_small) launch_pdl(k_sys_resample_small<2>, T.rs_small, SCAN_BLOCK, 0, st, P);
    else if (P.multinomial) launch_pdl(k_sys_resample<2, true>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<2>), st, P);
    else launch_pdl(k_sys_resample<2>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<2>), st, P);
    if (P.multinomial) {
      mark("k_multinomial_emit");
      k_multinomial_emit<<<grid_for(P.n, 256, ctx->sms), 256, 0, st>>>(P);
    }
  }
  if (evs) cudaEventRecord(evs[q], st);
  PCS_LAUNCH_CHECK();
  T.launches = q;
  return PCS_OK;
}

static bool g_attr_done = false;

static int set_attrs() {
  if (g_attr_done) return PCS_OK;
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_pc_step1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)S1_SMEM));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_pc_step1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)S1_SMEM));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_pc_step1<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)S1_SMEM_Q));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_pc_step1<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)S1_SMEM_Q));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_sys_resample<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(RsSmem<1>)));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_sys_resample<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(RsSmem<2>)));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_sys_resample<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(RsSmem<1>)));
  PCS_CUDA_TRY(cudaFuncSetAttribute(k_sys_resample<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(RsSmem<2>)));
  // one shared-memory carveout for every kernel of the frame: consecutive
  // kernels with different carveouts force an SM reconfiguration between them
  const void* fns[] = {(const void*)k_pc_step1<true>,  (const void*)k_pc_step1<false>,
                       (const void*)k_pc_step1<true, true>, (const void*)k_pc_step1<false, true>,
                       (const void*)k_pc_bins,
                       (const void*)k_pc_cells,         (const void*)k_sir_propagate_lik<0>,
                       (const void*)k_sir_propagate_lik<9>, (const void*)k_sir_propagate_lik<11>,
                       (const void*)k_sir_propagate_lik<15>, (const void*)k_sir_sum,
                       (const void*)k_sir_stats,        (const void*)k_sys_resample<1>,
                       (const void*)k_sys_resample<2>,  (const void*)k_sys_resample_small<1>,
                       (const void*)k_sys_resample_small<2>};
  for (const void* f : fns)
    PCS_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      (int)cudaSharedmemCarveoutMaxShared));
  g_attr_done = true;
  return PCS_OK;
}

static int track_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t H, int64_t W, i64 extra_ld,
                       void* stream);

int pcs_track_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t H, int64_t W, void* stream) {
  return track_begin(ctx, cfg, H, W, 0, stream);
}

// extra_ld: state slots after the n particles (the sharded filter's received
// boundary states)
static int track_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t H, int64_t W, i64 extra_ld,
                       void* stream) {
  PCS_CHECK_ARG(ctx && cfg, "bad arguments");
  PCS_CHECK_ARG(cfg->method == 0 || cfg->method == 1, "method must be 0 (SIR) or 1 (pcSIR)");
  // (32-bit particle indices in the fused kernels, with a chunk of headroom)
  PCS_CHECK_ARG(cfg->n_particles >= 1 && cfg->n_particles <= (i64)INT_MAX - 4096,
                "n_particles out of range");
  PCS_CHECK_ARG(H >= 1 && W >= 1, "bad frame shape");
  int r = check_spot(&cfg->spot);
  if (r) return r;
  if (cfg->method == 1) {
    r = check_grid(&cfg->grid);
    if (r) return r;
    PCS_CHECK_ARG(cfg->placement == 0 || cfg->placement == 1, "unknown placement");
    if ((double)cfg->grid.n_cols * (double)cfg->grid.n_rows > (double)TABLE_MAX) {
      pcs_set_last_error("grid exceeds the fused loop's cell ids (2^32 - 1 cells)");
      return PCS_E_CAPACITY;
    }
  }
  PCS_CHECK_ARG(cfg->dyn.dt > 0, "dt must be > 0");
  cudaStream_t st = S(stream);
  r = set_attrs();
  if (r) return r;
  track_release(ctx);
  TrackState& T = ctx->tr;
  T = TrackState();
  T.cfg = *cfg;
  const i64 n = cfg->n_particles;
  const i64 ld = ceil_div(n + extra_ld, 32) * 32;
  TrackParams& P = T.P;
  P.n = n;
  P.ld = ld;
  P.H = H;
  P.W = W;
  P.dyn = make_dyn(cfg->dyn.sigma_pos, cfg->dyn.sigma_vel, cfg->dyn.sigma_int, cfg->dyn.dt);
  P.spot = to_spot(&cfg->spot);
  P.grid = cfg->method == 1 ? to_grid(&cfg->grid) : Grid{0, 0, 1, 1, 1, 1};
  P.inv_lx = 1.0 / P.grid.lx;
  P.inv_ly = 1.0 / P.grid.ly;
  P.axx = make_axis(P.grid.ox, P.grid.lx, P.inv_lx, P.grid.ncols);
  P.axy = make_axis(P.grid.oy, P.grid.ly, P.inv_ly, P.grid.nrows);
  P.seed = cfg->seed;
  P.pk = philox_key(cfg->seed);
  P.frame0 = cfg->frame0;
  P.placement = cfg->placement;
  P.weighted = (cfg->method == 1 && cfg->placement == 0 && cfg->weighted_com) ? 1 : 0;
  P.idx_off = 0;
  P.n_global = n;
  P.slot_lo = 0;
  P.slot_cap = n;
  P.scan_mode = 0;
  P.method = cfg->method;
  PCS_CHECK_ARG(cfg->scheme == 0 || cfg->scheme == 1, "scheme must be 0 (systematic) or 1 (multinomial)");
  P.multinomial = cfg->scheme;
  P.cdf = nullptr;
  if (P.multinomial) PCS_SCRATCH(SL_TR_CDF, ld * sizeof(double), P.cdf);
  PCS_SCRATCH(SL_TR_BUF0, 5 * ld * sizeof(float), P.buf0);
  PCS_SCRATCH(SL_TR_BUF1, 5 * ld * sizeof(float), P.buf1);
  PCS_SCRATCH(SL_TR_ANC, ld * sizeof(int), P.anc);
  P.anc_out = P.anc;
  PCS_SCRATCH(SL_TR_CTL, sizeof(TrackCtl), P.ctl);
  PCS_SCRATCH(SL_FMAP, 128, P.fmap);
  P.ntiles = ceil_div(n, SCAN_TILE);
  // per-CTA aggregates of the resampler: one per CTA (<= one per RSS_TILE particles)
  const i64 nagg = std::max<i64>(P.ntiles, ceil_div(n, (i64)RSS_TILE));
  PCS_SCRATCH(SL_TR_TILES, P.ntiles * (2 * sizeof(u128) + sizeof(u32)) + nagg * sizeof(u128) + 64,
              P.tile_agg);
  P.tile_inc = P.tile_agg + P.ntiles;
  P.cta_agg = P.tile_inc + P.ntiles;
  P.tile_status = (u32*)(P.cta_agg + nagg);
  PCS_CUDA_TRY(cudaMemsetAsync(P.tile_status, 0, P.ntiles * sizeof(u32), st));
  {
    const double frac = cfg->threshold_fraction > 0.0 ? cfg->threshold_fraction : 1.0;
    PCS_CHECK_ARG(frac <= 1.0, "threshold_fraction must be in (0, 1]");
    P.thresh = frac * (double)n;   // the reference's threshold_fraction * n_particles
  }
  if (cfg->method == 0) {
    PCS_SCRATCH(SL_TR_LL, ld * sizeof(double), P.ll);
    PCS_SCRATCH(SL_TR_WPREV, ld * sizeof(float), P.wprev);
    P.pslot = nullptr;
  } else {
    PCS_SCRATCH(SL_TR_PSLOT, ld * sizeof(u32), P.pslot);
    P.ll = nullptr;
    P.wprev = nullptr;
    P.lltab = nullptr;
    P.G = HT_CAP;   // per-frame cell table: hashed slots (any grid up to 2^32 - 1 cells)
    T.cond = P.thresh < (double)n;   // threshold resampling: frames may carry prior weights
    if (T.cond) {
      PCS_SCRATCH(SL_TR_LL, ld * sizeof(double), P.ll);
      PCS_SCRATCH(SL_TR_WPREV, ld * sizeof(float), P.wprev);
      PCS_SCRATCH(SL_TR_LLTAB, P.G * sizeof(double), P.lltab);
    }
    if (!ctx->tab_cnt) {
      // keys, counts, then the float / exact cdf weights per slot
      PCS_CUDA_TRY(cudaMalloc(&ctx->tab_cnt, 2 * (size_t)HT_CAP * sizeof(u32)));
      PCS_CUDA_TRY(cudaMalloc(&ctx->tab_sum, 5 * (size_t)HT_CAP * (2 + TAB_LIMBS) * sizeof(u64)));
      // (the exact weights of the SUBW sub-window cells sit right in front of the
      // per-slot ones: a particle's cell code indexes both, code_wfix)
      PCS_CUDA_TRY(cudaMalloc(&ctx->wtab, (size_t)HT_CAP * (sizeof(float) + sizeof(u128)) + SUBW * sizeof(u128)));
      ctx->table_cells = HT_CAP;
      ctx->table_dirty = true;
    }
    // occupied-cell list + per-cell log-likelihood and count (k_pc_cells)
    if (!ctx->occ) PCS_CUDA_TRY(cudaMalloc(&ctx->occ, MAXM * (sizeof(u32) + sizeof(double) + sizeof(u32))));
    if (ctx->table_dirty) {
      PCS_CUDA_TRY(cudaMemsetAsync(ctx->tab_cnt, 0, (size_t)HT_CAP * sizeof(u32), st));
      PCS_CUDA_TRY(cudaMemsetAsync(ctx->tab_cnt + HT_CAP, 0xFF, (size_t)HT_CAP * sizeof(u32), st));
      PCS_CUDA_TRY(cudaMemsetAsync(ctx->tab_sum, 0, 5 * (size_t)HT_CAP * (2 + TAB_LIMBS) * sizeof(u64), st));
      ctx->table_dirty = false;
    }
    // compact per-frame tables of the step-1 sub-window cells (pslot codes < SUBW)
    PCS_SCRATCH(SL_TR_SUB, SUBW * (sizeof(double) + sizeof(float)), P.ltsub);
    P.wtsub = (float*)(P.ltsub + SUBW);
    P.wsub = (u128*)ctx->wtab;
    P.tab_cnt = ctx->tab_cnt;
    P.hkey = ctx->tab_cnt + HT_CAP;
    P.tab_sum = ctx->tab_sum;
    P.tab_lim = ctx->tab_sum + 5 * (size_t)HT_CAP * 2;
    P.wfix = P.wsub + SUBW;
    P.wtab = (float*)(P.wfix + HT_CAP);
    P.occ = ctx->occ;
    T.bins.ll = (double*)(ctx->occ + MAXM);
    T.bins.cnt = (u32*)(T.bins.ll + MAXM);
  }
  T.maxs = maxs_for(cfg->spot.halfwidth);
  // SIR reductions: >= 16 particles per thread (few int128 partials per atomic
  // target at c2 sizes), 2..8 CTAs per SM
  T.red_grid = (int)std::min<i64>((i64)ctx->sms * 8,
                                  std::max<i64>((i64)ctx->sms * 2, ceil_div(n, (i64)256 * 16)));
  {
    // SIR propagate + likelihood: every resident CTA stages the frame region
    // once and strides over the particles (no later waves re-staging it)
    const void* f = T.maxs == 9    ? (const void*)k_sir_propagate_lik<9>
                    : T.maxs == 11 ? (const void*)k_sir_propagate_lik<11>
                    : T.maxs == 15 ? (const void*)k_sir_propagate_lik<15>
                                   : (const void*)k_sir_propagate_lik<0>;
    int per_sm = 1;
    PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 256, 0));
    T.prop_grid = (int)std::min<i64>((i64)grid_for(n, 256, ctx->sms, 8),
                                     (i64)ctx->sms * std::max(per_sm, 1));
    // dynamic chunks of 2048 when every CTA gets >= 8 of them; below that a
    // plain grid stride (c1/c2 sizes: the tickets would not pay)
    P.sir_chunk = (n >= (i64)T.prop_grid * 8 * 2048) ? 2048 : 0;
  }
  T.s1_grid = (int)std::min<i64>((i64)ctx->sms * S1_CTAS_PER_SM, std::max<i64>(1, ceil_div(n, (i64)S1_THREADS * 4)));
  T.cells_grid = ctx->sms * 4;
  T.s1_pow2 = cfg->method == 1 && grid_pow2(P.grid.ox, P.grid.lx, P.grid.oy, P.grid.ly);
  P.ht_shift = -1;   // bit-slice table hash when the grid has 2^k columns
  if (getenv("PCS_HT_MULT") == nullptr)
    for (int b = 0; b < 31; ++b)
      if (P.grid.ncols == ((i64)1 << b)) P.ht_shift = b;
  {
    // equal tile counts per warp: tile = ceil(per_warp / ceil(per_warp / S1_MAX_WT))
    const i64 per_warp = ceil_div(n, (i64)T.s1_grid * S1_WARPS);
    const i64 tpw = ceil_div(per_warp, (i64)S1_MAX_WT);
    P.s1_tile = (int)std::max<i64>(32, ceil_div(per_warp, tpw));
  }
  {
    // k_sys_resample has a grid barrier: every CTA must be co-resident
    int per_sm = 0;
    if (cfg->method == 1)
      PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sys_resample<1>, SCAN_BLOCK,
                                                                 sizeof(RsSmem<1>)));
    else
      PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sys_resample<2>, SCAN_BLOCK,
                                                                 sizeof(RsSmem<2>)));
    T.rs_grid = (int)std::min<i64>((i64)ctx->sms * std::max(per_sm, 1), ceil_div(n, (i64)RS_TILE));
    T.rs_grid2 = T.rs_grid;
    if (T.cond) {   // pcSIR frames with prior weights resample per particle
      int per2 = 0;
      PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_sys_resample<2>, SCAN_BLOCK,
                                                                 sizeof(RsSmem<2>)));
      T.rs_grid2 = (int)std::min<i64>((i64)ctx->sms * std::max(per2, 1), ceil_div(n, (i64)RS_TILE));
    }
    // small N: one RSS_TILE tile per CTA when all those CTAs are co-resident
    int per_small = 0;
    if (cfg->method == 1)
      PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_small, k_sys_resample_small<1>,
                                                                 SCAN_BLOCK, 0));
    if (cfg->method == 0 || T.cond) {
      int per2 = 0;
      PCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_sys_resample_small<2>,
                                                                 SCAN_BLOCK, 0));
      per_small = (cfg->method == 0) ? per2 : std::min(per_small, per2);
    }
    const i64 g_small = ceil_div(n, (i64)RSS_TILE);
    T.rs_small = (g_small <= (i64)ctx->sms * per_small && getenv("PCS_NO_RS_SMALL") == nullptr)
                     ? (int)g_small : 0;
  }
  // initial cloud (state.py:164-175) and identity ancestors
  pcs_init_t init = cfg->init;
  r = pcs_init_particles(&init, cfg->seed, 0, n, P.buf0, ld, stream);
  if (r) return r;
  k_iota<<<grid_for(n, 256, ctx->sms), 256, 0, st>>>(P.anc, n);
  k_ctl_init<<<1, 1, 0, st>>>(P.ctl, init.center[0], init.center[1]);
  PCS_LAUNCH_CHECK();
  T.k = 0;
  T.active = true;
  if (cfg->use_graph) {
    // capture one frame on the private stream; replays read everything from the control block
    PCS_CUDA_TRY(cudaStreamSynchronize(st));
    PCS_CUDA_TRY(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
    int er = enqueue_frame(ctx, ctx->cap);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctx->cap, &g);
    if (er) return er;
    PCS_CUDA_TRY(e);
    T.graph = g;
    PCS_CUDA_TRY(cudaGraphInstantiate(&T.exec, g, 0));
  }
  return PCS_OK;
}

// TMA descriptor of a batch of frames [K][H][W] float32 (boxes FMAP_BX x
// FMAP_BY x 1), written to the track's device slot; 0 if unavailable (the
// kernels then stage with plain loads)
static PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
static int frame_map(TrackState& T, const float* frames, i64 nframes, cudaStream_t st) {
  static const bool disabled = getenv("PCS_NO_TMA") != nullptr;
  if (disabled) return 0;
  if (!g_encode_tiled) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return 0;
    g_encode_tiled = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const i64 W = T.P.W, H = T.P.H;
  if (!T.P.fmap || nframes < 1 || (W * 4) % 16 || ((uintptr_t)frames) % 16) return 0;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)nframes};
  cuuint64_t strides[2] = {(cuuint64_t)(W * 4), (cuuint64_t)(W * H * 4)};
  cuuint32_t box[3] = {FMAP_BX, FMAP_BY, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (g_encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)frames, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 0;
  if (cudaMemcpyAsync((void*)T.P.fmap, &m, sizeof(m), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return 0;
  return 1;
}

int pcs_track_steps(pcs_ctx* ctx, const float* frames, int64_t k0, int64_t k1, double* est,
                    double* ess, uint8_t* res, int64_t* occ, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active, "no active track (call pcs_track_begin)");
  PCS_CHECK_ARG(frames && est && ess && res && occ, "bad arguments");
  PCS_CHECK_ARG(k0 == ctx->tr.k && k1 >= k0, "frames must be stepped in order");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  const int fm = frame_map(T, frames, k1 - k0, st);
  k_ctl_io<<<1, 1, 0, st>>>(T.P.ctl, frames, k0, k0, k1, est, ess, res, (i64*)occ, fm);
  PCS_LAUNCH_CHECK();
  for (i64 k = k0; k < k1; ++k) {
    if (T.exec && k > 0) {
      PCS_CUDA_TRY(cudaGraphLaunch(T.exec, st));
    } else {   // (the first frame of a track is launched directly: its own step-1 form)
      int r = enqueue_frame(ctx, st, nullptr, k == 0);
      if (r) return r;
    }
  }
  T.k = k1;
  return PCS_OK;
}

int pcs_track_steps_timed(pcs_ctx* ctx, const float* frames, int64_t k0, int64_t k1, double* est,
                          double* ess, uint8_t* res, int64_t* occ, double* kernel_ms,
                          int32_t max_kernels, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active, "no active track (call pcs_track_begin)");
  PCS_CHECK_ARG(frames && est && ess && res && occ && kernel_ms && max_kernels >= 8,
                "bad arguments");
  PCS_CHECK_ARG(k0 == ctx->tr.k && k1 >= k0, "frames must be stepped in order");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  const int fm = frame_map(T, frames, k1 - k0, st);
  k_ctl_io<<<1, 1, 0, st>>>(T.P.ctl, frames, k0, k0, k1, est, ess, res, (i64*)occ, fm);
  PCS_LAUNCH_CHECK();
  const int NE = TrackState::MAX_LAUNCHES + 1;
  cudaEvent_t evs[NE];
  for (int i = 0; i < NE; ++i) PCS_CUDA_TRY(cudaEventCreate(&evs[i]));
  for (int i = 0; i < max_kernels; ++i) kernel_ms[i] = 0.0;
  int r = PCS_OK;
  for (i64 k = k0; k < k1 && r == PCS_OK; ++k) {
    r = enqueue_frame(ctx, st, evs, k == 0);
    if (r) break;
    cudaError_t e = cudaEventSynchronize(evs[T.launches]);
    if (e != cudaSuccess) {
      pcs_set_last_error(cudaGetErrorString(e));
      r = PCS_E_CUDA;
      break;
    }
    for (int q = 0; q < std::min(T.launches, (int)max_kernels); ++q) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, evs[q], evs[q + 1]);
      kernel_ms[q] += ms;
    }
  }
  for (int i = 0; i < NE; ++i) cudaEventDestroy(evs[i]);
  if (r == PCS_OK) T.k = k1;
  return r;
}

const char* pcs_track_kernel_name(pcs_ctx* ctx, int32_t i) {
  if (!ctx || i < 0 || i >= ctx->tr.launches || i >= TrackState::MAX_LAUNCHES) return "";
  return ctx->tr.names[i] ? ctx->tr.names[i] : "";
}

int pcs_track_end(pcs_ctx* ctx, pcs_track_result_t* result, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && result, "bad arguments");
  cudaStream_t st = S(stream);
  TrackCtl h;
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, ctx->tr.P.ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  result->flags = h.flags;
  result->first_bad_frame = (h.first_bad == INT_MAX) ? -1 : h.first_bad;
  result->likelihood_evals = h.evals;
  if (h.flags & PCS_FLAG_CAPACITY) ctx->table_dirty = true;
  if (h.flags & PCS_FLAG_CAPACITY) return PCS_E_CAPACITY;
  return PCS_OK;
}

int pcs_track(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, const float* frames, int64_t K,
              int64_t H, int64_t W, double* est, double* ess, uint8_t* res, int64_t* occ,
              pcs_track_result_t* result, void* stream) {
  PCS_CHECK_ARG(K >= 1, "need at least one frame");
  int r = pcs_track_begin(ctx, cfg, H, W, stream);
  if (r) return r;
  r = pcs_track_steps(ctx, frames, 0, K, est, ess, res, occ, stream);
  if (r) return r;
  return pcs_track_end(ctx, result, stream);
}

int pcs_track_launches_per_step(pcs_ctx* ctx) { return ctx ? ctx->tr.launches : 0; }

// ---------------------------------------------------------------------------
// batched multi-target pcSIR (config 4): one CTA per target per frame
// ---------------------------------------------------------------------------
int pcs_mt_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t n_targets,
                 const double* centers, int64_t target_offset, int64_t n_frames, int64_t H,
                 int64_t W, void* stream) {
  PCS_CHECK_ARG(ctx && cfg && centers && n_targets >= 1 && n_frames >= 1, "bad arguments");
  PCS_CHECK_ARG(cfg->method == 1, "multi-target filter is pcSIR");
  PCS_CHECK_ARG(cfg->n_particles >= 1 && (double)cfg->n_particles * n_targets < 2.0e9,
                "too many particles for 32-bit ancestors");
  // a cell gets <= 2 digit additions per warp per tile and the digits are never
  // flushed inside a frame: <= MT_MAX_TILES tiles keep them exact
  PCS_CHECK_ARG(cfg->n_particles <= (i64)MT_MAX_TILES * MT_TILE,
                "too many particles per target for the multi-target kernel");
  int r = check_spot(&cfg->spot);
  if (r) return r;
  r = check_grid(&cfg->grid);
  if (r) return r;
  PCS_CHECK_ARG((double)cfg->grid.n_cols * cfg->grid.n_rows < 4.0e9, "grid exceeds 32-bit cells");
  cudaStream_t st = S(stream);
  static bool attr = false;
  if (!attr) {
    const void* fns[] = {(const void*)k_mt_frame<0, false>, (const void*)k_mt_frame<9, false>,
                         (const void*)k_mt_frame<11, false>, (const void*)k_mt_frame<15, false>,
                         (const void*)k_mt_frame<0, true>, (const void*)k_mt_frame<9, true>,
                         (const void*)k_mt_frame<11, true>, (const void*)k_mt_frame<15, true>};
    for (const void* f : fns) {
      PCS_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)MT_SMEM));
      PCS_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        (int)cudaSharedmemCarveoutMaxShared));
    }
    attr = true;
  }
  MtState& M = ctx->mt;
  M = MtState();
  MtParams& P = M.P;
  const i64 n = cfg->n_particles, T = n_targets, ld = n * T;
  P.T = T;
  P.n = n;
  P.ld = ld;
  P.H = H;
  P.W = W;
  P.dyn = make_dyn(cfg->dyn.sigma_pos, cfg->dyn.sigma_vel, cfg->dyn.sigma_int, cfg->dyn.dt);
  P.spot = to_spot(&cfg->spot);
  P.grid = to_grid(&cfg->grid);
  P.inv_lx = 1.0 / P.grid.lx;
  P.inv_ly = 1.0 / P.grid.ly;
  P.pow2 = grid_pow2(P.grid.ox, P.grid.lx, P.grid.oy, P.grid.ly) ? 1 : 0;
  P.seed = cfg->seed;
  P.tgt_off = target_offset;
  P.frame0 = cfg->frame0;
  P.placement = cfg->placement;
  P.K = n_frames;
  PCS_CHECK_ARG(cfg->scheme == 0 || cfg->scheme == 1, "scheme must be 0 (systematic) or 1 (multinomial)");
  PCS_CHECK_ARG(!cfg->weighted_com, "the multi-target kernel places dummies at the unweighted centre of mass");
  const double frac = cfg->threshold_fraction > 0.0 ? cfg->threshold_fraction : 1.0;
  PCS_CHECK_ARG(frac <= 1.0, "threshold_fraction must be in (0, 1]");
  P.thresh = frac * (double)n;   // the reference's threshold_fraction * n_particles
  P.multinomial = cfg->scheme;
  P.wprev = nullptr;
  P.ll = nullptr;
  P.cdf = nullptr;
  if (P.thresh < (double)n) {    // frames may carry prior weights
    PCS_SCRATCH(SL_MT_WPREV, ld * sizeof(float), P.wprev);
    PCS_SCRATCH(SL_MT_LL, ld * sizeof(double), P.ll);
  }
  if (P.multinomial) PCS_SCRATCH(SL_MT_CDF, ld * sizeof(double), P.cdf);
  PCS_SCRATCH(SL_MT_BUF0, 5 * ld * sizeof(float), P.buf0);
  PCS_SCRATCH(SL_MT_BUF1, 5 * ld * sizeof(float), P.buf1);
  PCS_SCRATCH(SL_MT_ANC, ld * sizeof(int), P.anc);
  PCS_SCRATCH(SL_MT_PSLOT, ld * sizeof(u32), P.pslot);
  PCS_SCRATCH(SL_MT_TGT, T * sizeof(MtTarget), P.tgt);
  PCS_SCRATCH(SL_MT_HASH, T * MT_HCAP * sizeof(MtHash), P.hash);
  PCS_SCRATCH(SL_MT_OUT, T * n_frames * (5 * sizeof(double) + sizeof(double) + sizeof(i64) + 1) + 64,
              P.out_est);
  P.out_ess = P.out_est + T * n_frames * 5;
  P.out_occ = (i64*)(P.out_ess + T * n_frames);
  P.out_res = (unsigned char*)(P.out_occ + T * n_frames);
  PCS_CUDA_TRY(cudaMemsetAsync(P.hash, 0, T * MT_HCAP * sizeof(MtHash), st));
  std::vector<MtTarget> h(T);
  for (i64 t = 0; t < T; ++t) {
    h[t].center[0] = centers[t * 5 + 0];
    h[t].center[1] = centers[t * 5 + 1];
    h[t].flags = 0;
    h[t].first_bad = INT_MAX;
    h[t].evals = 0;
    h[t].prior = 0;
    h[t].span = 0;
    pcs_init_t init = cfg->init;
    for (int c = 0; c < 5; ++c) init.center[c] = centers[t * 5 + c];
    const u64 seed_t = cfg->seed + (u64)(target_offset + t) * MT_KEY_STEP;
    // each target's SoA slice: component c at c*ld + t*n
    InitSpecDev d = to_init(&init);
    k_init<<<grid_for(n, 256, ctx->sms), 256, 0, st>>>(d, seed_t, 0, n, P.buf0 + t * n, ld);
  }
  k_iota_mod<<<grid_for(ld, 256, ctx->sms), 256, 0, st>>>(P.anc, ld, n);
  PCS_CUDA_TRY(cudaMemcpyAsync(P.tgt, h.data(), T * sizeof(MtTarget), cudaMemcpyHostToDevice, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));   // h goes out of scope
  PCS_LAUNCH_CHECK();
  M.maxs = maxs_for(cfg->spot.halfwidth);
  M.k = 0;
  M.active = true;
  return PCS_OK;
}

int pcs_mt_step(pcs_ctx* ctx, const float* frame, int64_t k, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->mt.active && frame, "bad arguments");
  PCS_CHECK_ARG(k == ctx->mt.k && k < ctx->mt.P.K, "frames must be stepped in order");
  MtState& M = ctx->mt;
  M.P.frame = frame;
  M.P.k = k;
  cudaStream_t st = S(stream);
  const unsigned grid = (unsigned)M.P.T;
  const bool gen = M.P.thresh < (double)M.P.n || M.P.multinomial;
#define PCS_MT_LAUNCH(S)                                                       \
  (gen ? k_mt_frame<S, true><<<grid, MT_THREADS, MT_SMEM, st>>>(M.P)           \
       : k_mt_frame<S, false><<<grid, MT_THREADS, MT_SMEM, st>>>(M.P))
  switch (M.maxs) {
    case 9: PCS_MT_LAUNCH(9); break;
    case 11: PCS_MT_LAUNCH(11); break;
    case 15: PCS_MT_LAUNCH(15); break;
    default: PCS_MT_LAUNCH(0);
  }
#undef PCS_MT_LAUNCH
  PCS_LAUNCH_CHECK();
  M.k = k + 1;
  return PCS_OK;
}

// copy the outputs: est[T][K][5], ess[T][K], resampled[T][K], occupied[T][K];
// flags[T], evals[T], first_bad[T] (host arrays; NULL skips)
int pcs_mt_results(pcs_ctx* ctx, double* est, double* ess, uint8_t* res, int64_t* occ,
                   uint32_t* flags, int64_t* evals, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->mt.active, "bad arguments");
  cudaStream_t st = S(stream);
  const MtParams& P = ctx->mt.P;
  const i64 TK = P.T * P.K;
  if (est) PCS_CUDA_TRY(cudaMemcpyAsync(est, P.out_est, TK * 5 * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (ess) PCS_CUDA_TRY(cudaMemcpyAsync(ess, P.out_ess, TK * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (res) PCS_CUDA_TRY(cudaMemcpyAsync(res, P.out_res, TK, cudaMemcpyDeviceToHost, st));
  if (occ) PCS_CUDA_TRY(cudaMemcpyAsync(occ, P.out_occ, TK * sizeof(i64), cudaMemcpyDeviceToHost, st));
  std::vector<MtTarget> h(P.T);
  PCS_CUDA_TRY(cudaMemcpyAsync(h.data(), P.tgt, P.T * sizeof(MtTarget), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  for (i64 t = 0; t < P.T; ++t) {
    if (flags) flags[t] = h[t].flags;
    if (evals) evals[t] = h[t].evals;
  }
  return PCS_OK;
}

// ---------------------------------------------------------------------------
// particle-sharded giant filter (config 5): one rank's side of each phase
// ---------------------------------------------------------------------------
int pcs_shard_begin(pcs_ctx* ctx, const pcs_track_cfg_t* cfg, int64_t H, int64_t W, int32_t rank,
                    int32_t world, int64_t n_global, int64_t wcap, int64_t bcap, void* stream) {
  PCS_CHECK_ARG(ctx && cfg && cfg->method == 1, "sharded filter is pcSIR only");
  PCS_CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
  PCS_CHECK_ARG(n_global == (int64_t)world * cfg->n_particles, "n_global must be world x n_local");
  PCS_CHECK_ARG(wcap >= 1 && bcap >= 1 && bcap <= cfg->n_particles, "bad exchange capacities");
  PCS_CHECK_ARG(cfg->scheme == 0 || cfg->scheme == 1, "scheme must be 0 (systematic) or 1 (multinomial)");
  const double frac = cfg->threshold_fraction > 0.0 ? cfg->threshold_fraction : 1.0;
  PCS_CHECK_ARG(frac <= 1.0, "threshold_fraction must be in (0, 1]");
  // systematic: boundary states from / to the two neighbours (2 bcap extra
  // particles); multinomial: up to bcap answered requests from every rank
  const i64 extra = cfg->scheme ? (i64)world * bcap : 2 * bcap;
  pcs_track_cfg_t c = *cfg;
  c.use_graph = 0;
  int r = track_begin(ctx, &c, H, W, extra, stream);
  if (r) return r;
  TrackState& T = ctx->tr;
  TrackParams& P = T.P;
  P.idx_off = (i64)rank * cfg->n_particles;
  P.n_global = n_global;
  P.thresh = frac * (double)n_global;   // threshold_fraction x the global particle count
  P.sharded = 1;
  P.slot_cap = cfg->n_particles + 2 * bcap;
  PCS_SCRATCH(SL_SHARD_ANC, P.slot_cap * sizeof(int), P.anc_out);
  T.shard_bnd = nullptr;
  T.shard_cnt = nullptr;
  if (cfg->scheme) {
    PCS_SCRATCH(SL_SHARD_BND, world * sizeof(double), T.shard_bnd);
    PCS_SCRATCH(SL_SHARD_CNT, 2 * world * sizeof(u32), T.shard_cnt);
    PCS_CUDA_TRY(cudaMemsetAsync(T.shard_cnt, 0, 2 * world * sizeof(u32), S(stream)));
  }
  T.shard_rank = rank;
  T.shard_world = world;
  T.shard_wcap = wcap;
  T.shard_bcap = bcap;
  // the initial cloud uses the global particle index as the Philox counter
  pcs_init_t init = cfg->init;
  r = pcs_init_particles(&init, cfg->seed, P.idx_off, P.n, P.buf0, P.ld, stream);
  if (r) return r;
  return PCS_OK;
}

int pcs_shard_step1(pcs_ctx* ctx, const float* frame, int64_t k, double* est, double* ess,
                    uint8_t* res, int64_t* occ, int64_t* box, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && frame && box, "bad arguments");
  PCS_CHECK_ARG(k == ctx->tr.k, "frames must be stepped in order");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  k_ctl_io<<<1, 1, 0, st>>>(T.P.ctl, frame, k, k, k + 1, est, ess, res, (i64*)occ);
  if (k == 0) {   // (the track's first frame: the queued form, as enqueue_frame)
    if (T.s1_pow2) k_pc_step1<true, true><<<T.s1_grid, S1_THREADS, S1_SMEM_Q, st>>>(T.P);
    else k_pc_step1<false, true><<<T.s1_grid, S1_THREADS, S1_SMEM_Q, st>>>(T.P);
  } else {
    if (T.s1_pow2) k_pc_step1<true><<<T.s1_grid, S1_THREADS, S1_SMEM, st>>>(T.P);
    else k_pc_step1<false><<<T.s1_grid, S1_THREADS, S1_SMEM, st>>>(T.P);
  }
  k_shard_bbox<<<1, 1024, 0, st>>>(T.P, (i64*)box);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_shard_export(pcs_ctx* ctx, const int64_t* box, int64_t* limbs, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && box && limbs, "bad arguments");
  const TrackState& T = ctx->tr;
  k_shard_export<<<grid_for(T.shard_wcap, 256, ctx->sms), 256, 0, S(stream)>>>(
      T.P, (const i64*)box, T.shard_wcap, (i64*)limbs);
  k_shard_reset<<<1, 1024, 0, S(stream)>>>(T.P);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_shard_import_bins(pcs_ctx* ctx, const int64_t* box, const int64_t* limbs, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && box && limbs, "bad arguments");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  k_shard_import<<<grid_for(T.shard_wcap, 256, ctx->sms), 256, 0, st>>>(
      T.P, (const i64*)box, T.shard_wcap, (const i64*)limbs);
  k_pc_cells<<<T.cells_grid, CELLS_BLOCK, 0, st>>>(T.P, T.bins);
  k_pc_bins<<<1, BINS_BLOCK, 0, st>>>(T.P, T.bins);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_shard_total(pcs_ctx* ctx, int64_t* total, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && total, "bad arguments");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  TrackParams Q = T.P;
  Q.scan_mode = 1;
  launch_pdl(k_sys_resample<1>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<1>), st, Q);
  if (T.cond) launch_pdl(k_sys_resample<2>, T.rs_grid2, SCAN_BLOCK, sizeof(RsSmem<2>), st, Q);
  k_shard_total<<<1, 32, 0, st>>>(Q, T.rs_grid, T.rs_grid2, (i64*)total);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_shard_emit(pcs_ctx* ctx, const int64_t* totals, float* send_prev, float* send_next,
                   void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && totals && send_prev && send_next, "bad arguments");
  PCS_CHECK_ARG(!ctx->tr.P.multinomial, "multinomial resampling exchanges through pcs_shard_route");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  k_shard_ranges<<<1, 32, 0, st>>>(T.P, (const i64*)totals, T.shard_rank, T.shard_world,
                                   T.shard_bcap, 0, nullptr);
  TrackParams Q = T.P;
  Q.scan_mode = 2;
  launch_pdl(k_sys_resample<1>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<1>), st, Q);
  if (T.cond) launch_pdl(k_sys_resample<2>, T.rs_grid2, SCAN_BLOCK, sizeof(RsSmem<2>), st, Q);
  k_shard_pack<<<grid_for(T.P.n, 256, ctx->sms), 256, 0, st>>>(T.P, T.shard_rank, send_prev,
                                                              send_next, T.shard_bcap);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

int pcs_shard_unpack(pcs_ctx* ctx, const float* recv_prev, const float* recv_next, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && recv_prev && recv_next, "bad arguments");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  k_shard_unpack<<<grid_for(T.shard_bcap, 256, ctx->sms), 256, 0, st>>>(T.P, recv_prev, recv_next,
                                                                        T.shard_bcap);
  PCS_LAUNCH_CHECK();
  T.k += 1;
  return PCS_OK;
}

// frames with prior weights (ESS threshold): stage 0 -> out[1] local max
// log-weight; stage 1 (in = reduced max) -> out[3] normaliser limbs; stage 2
// (in = reduced normaliser) -> out[18] estimate / ESS limbs, out_mm[2] weight
// range; stage 3 (in = reduced limbs, in_mm = reduced range) finalises the
// frame. Neutral values / no-ops on frames without prior weights.
int pcs_shard_prior(pcs_ctx* ctx, int32_t stage, const int64_t* in, const int64_t* in_mm,
                    int64_t* out, int64_t* out_mm, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && ctx->tr.P.sharded && stage >= 0 && stage <= 3,
                "bad arguments");
  PCS_CHECK_ARG((stage == 0 || in) && (stage < 3 ? out != nullptr : in_mm != nullptr) &&
                    (stage != 2 || out_mm), "bad arguments");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  if (!T.cond) return PCS_OK;   // threshold 1: no frame carries prior weights
  TrackParams& P = T.P;
  if (stage > 0) k_shard_prior_in<<<1, 32, 0, st>>>(P, stage - 1, (const i64*)in, (const i64*)in_mm);
  if (stage == 0) k_pc_prior_ll<<<T.red_grid, 256, 0, st>>>(P);
  if (stage == 1) k_sir_sum<<<T.red_grid, 256, 0, st>>>(P);
  if (stage == 2) k_sir_stats<<<T.red_grid, 256, 0, st>>>(P);
  if (stage < 3) k_shard_prior_out<<<1, 32, 0, st>>>(P, stage, (i64*)out, (i64*)out_mm);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// multinomial: exact rank prefix and boundary cdf values, the rank's part of
// the global cdf, local ancestors and the requests to the other ranks
// (req int32 [world][1 + bcap], count first)
int pcs_shard_route(pcs_ctx* ctx, const int64_t* totals, int32_t* req, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && totals && req, "bad arguments");
  PCS_CHECK_ARG(ctx->tr.P.multinomial, "systematic resampling exchanges through pcs_shard_emit");
  cudaStream_t st = S(stream);
  TrackState& T = ctx->tr;
  k_shard_ranges<<<1, 32, 0, st>>>(T.P, (const i64*)totals, T.shard_rank, T.shard_world,
                                   T.shard_bcap, 1, T.shard_bnd);
  TrackParams Q = T.P;
  Q.scan_mode = 2;
  launch_pdl(k_sys_resample<1, true>, T.rs_grid, SCAN_BLOCK, sizeof(RsSmem<1>), st, Q);
  if (T.cond) launch_pdl(k_sys_resample<2, true>, T.rs_grid2, SCAN_BLOCK, sizeof(RsSmem<2>), st, Q);
  k_shard_route<<<grid_for(T.P.n, 256, ctx->sms), 256, 0, st>>>(
      T.P, T.shard_rank, T.shard_world, T.shard_bnd, (int*)req, T.shard_cnt, T.shard_bcap);
  k_shard_route_fin<<<1, 256, 0, st>>>(T.P, T.shard_world, (int*)req, T.shard_cnt,
                                       T.shard_cnt + T.shard_world, T.shard_bcap);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// multinomial: answer the gathered requests (req_in int32 [world][1 + bcap])
// with the ancestors' states (resp float32 [world][5 * bcap])
int pcs_shard_serve(pcs_ctx* ctx, const int32_t* req_in, float* resp, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && ctx->tr.P.multinomial && req_in && resp, "bad arguments");
  TrackState& T = ctx->tr;
  const i64 total = (i64)T.shard_world * T.shard_bcap;
  k_shard_serve<<<grid_for(total, 256, ctx->sms), 256, 0, S(stream)>>>(
      T.P, T.shard_rank, T.shard_world, (const int*)req_in, resp, T.shard_bcap);
  PCS_LAUNCH_CHECK();
  return PCS_OK;
}

// multinomial: install the answered states (resp_in float32 [world][5 * bcap]);
// the frame is complete
int pcs_shard_install(pcs_ctx* ctx, const float* resp_in, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && ctx->tr.P.multinomial && resp_in, "bad arguments");
  TrackState& T = ctx->tr;
  const i64 total = (i64)T.shard_world * T.shard_bcap;
  k_shard_install<<<grid_for(total, 256, ctx->sms), 256, 0, S(stream)>>>(
      T.P, T.shard_rank, T.shard_world, resp_in, T.shard_cnt + T.shard_world, T.shard_bcap);
  PCS_LAUNCH_CHECK();
  T.k += 1;
  return PCS_OK;
}

int pcs_track_debug(pcs_ctx* ctx, int64_t* out16, void* stream) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && out16, "bad arguments");
  cudaStream_t st = S(stream);
  TrackCtl h;
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, ctx->tr.P.ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < 16; ++i) out16[i] = h.dbg[i];
  return PCS_OK;
}

int pcs_track_info(pcs_ctx* ctx, int64_t* out, int32_t n, void* stream) {
  PCS_CHECK_ARG(ctx && out && n >= 12, "bad arguments");
  PCS_CHECK_ARG(ctx->tr.P.ctl, "no track has been started");
  const TrackState& T = ctx->tr;
  const TrackParams& P = T.P;
  cudaStream_t st = S(stream);
  TrackCtl h;
  PCS_CUDA_TRY(cudaMemcpyAsync(&h, P.ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCS_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i) out[i] = 0;
  out[0] = T.s1_grid;
  out[1] = P.s1_tile;
  out[2] = (T.s1_grid > 0 && P.s1_tile > 0) ? ceil_div(ceil_div(P.n, (i64)P.s1_tile), (i64)T.s1_grid * S1_WARPS) : 0;
  out[3] = T.rs_small ? T.rs_small : T.rs_grid;
  out[4] = T.rs_small ? 1 : (T.rs_grid > 0 ? ceil_div(ceil_div(P.n, (i64)RS_TILE), (i64)T.rs_grid) : 0);
  out[5] = P.sir_chunk;
  out[6] = h.s1_mid_flush;
  out[7] = h.max_occ;
  out[8] = MAXM;
  out[9] = S1_CELL_FLUSH;
  out[10] = T.prop_grid;
  out[11] = T.launches;
  return PCS_OK;
}

int pcs_track_states(pcs_ctx* ctx, float** states, int64_t* ld) {
  PCS_CHECK_ARG(ctx && ctx->tr.active && states && ld, "bad arguments");
  // frame k reads buf[k&1] and writes buf[(k+1)&1]
  *states = (ctx->tr.k & 1) ? ctx->tr.P.buf1 : ctx->tr.P.buf0;
  *ld = ctx->tr.P.ld;
  return PCS_OK;
}

}  // extern "C"
