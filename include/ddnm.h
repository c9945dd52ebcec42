/*
 * ddnm.h -- C ABI of the B200-native batched DD NM-ROM-HR online solve.
 *
 * The reference (arxiv 2305.15163, /root/reference/pkg/src/ddrom) has no FFI:
 * its hot path is the Python call chain
 *     driver.solve_rom            driver.py:554-597
 *       -> build_problem          driver.py:356-436
 *       -> init_guess             driver.py:442-458 (RbfInitializer.query
 *                                 driver.py:82-90, multiplier_least_squares
 *                                 driver.py:461-471)
 *       -> sqp.iterate            sqp.py:230-299
 *            -> eval_gradients    sqp.py:117-146
 *            -> assemble_and_solve_kkt  sqp.py:162-208
 * Each entry point below replaces one of those calls for a whole batch of
 * parameters mu = (a, lambda) at once; the Python package
 * paper_2305_15163_b200 binds them with ctypes.
 *
 * Conventions: plain pointers and sizes, no torch types.  Host arrays are
 * caller-owned, row-major, FP64, indices int64 (the reference's dtypes).
 * One context per GPU; a context is not thread-safe; it owns one CUDA stream
 * and all device buffers.  Every function returns 0 on success or a negative
 * DDNM_E* code; ddnm_last_error() describes the most recent failure on the
 * calling thread.
 */
#ifndef DDNM_H
#define DDNM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDNM_ABI_VERSION 2

/* return codes */
#define DDNM_OK 0
#define DDNM_EINVAL (-1)       /* bad argument / shape (reference: ValueError) */
#define DDNM_ECUDA (-2)        /* CUDA runtime failure                          */
#define DDNM_EUNSUPPORTED (-3) /* latent dims / sizes without a compiled kernel */
#define DDNM_ENOMEM (-4)
#define DDNM_EFORMAT (-5)      /* malformed binio / instance file (reference: FormatError) */

/* per-mu solve status (reference: SqpResult.failure_reason / exceptions) */
#define DDNM_STATUS_OK 0           /* loop ended on tol or max_iter (sqp.py:255)   */
#define DDNM_STATUS_LINE_SEARCH 1  /* "line_search" failure, best iterate (sqp.py:275-293) */
#define DDNM_STATUS_KKT_SINGULAR 2 /* ConvergenceError from the KKT (sqp.py:199-207) */
#define DDNM_STATUS_LSTSQ_RANK 3   /* multiplier least squares rank deficient:
                                      K is then singular too (driver.py:461-471)   */

/* reduction-map kinds (RomInstance.interior_maps / interface_maps) */
#define DDNM_MAP_AUTOENCODER 0     /* sparse shallow decoder, autoencoder.py:99-174 */
#define DDNM_MAP_LINEAR 1          /* POD LinearMap, pod.py:67-97                   */

#define DDNM_ACT_SWISH 0           /* autoencoder.py:31-45 */
#define DDNM_ACT_SIGMOID 1

/* coupling of the interface latents (RomInstance.constraint_mode) */
#define DDNM_CON_WFPC 0            /* weak FOM-port: C A_i g^Gamma(x_Gamma), driver.py:366-373 */
#define DDNM_CON_SRPC 1            /* strong ROM-port: Ahat_i x_Gamma, driver.py:374-378      */

/* One decoder.  AUTOENCODER: g = (W2 act(W1 x + b1)) * scale + shift with W2 a
 * CSR matrix [n_out x n_hidden] in storage (= accumulation) order
 * (hyper.py:163-197).  LINEAR: g = Phi x, Phi = W1 [n_out x latent]. */
typedef struct {
  int32_t n_out;
  int32_t n_hidden;          /* AUTOENCODER only */
  const double* W1;          /* [n_hidden][latent] or Phi [n_out][latent] */
  const double* b1;          /* [n_hidden] */
  const int64_t* indptr;     /* [n_out + 1] */
  const int64_t* indices;    /* [nnz] hidden index per entry */
  const double* data;        /* [nnz] */
  const double* scale;       /* [n_out] */
  const double* shift;       /* [n_out] */
} ddnm_decoder;

/* One subdomain block as build_problem instantiates it (driver.py:360-435):
 * interior decoder restricted to the HR outputs `io` (extract_subnet,
 * hyper.py:200-222, or LinearMap.restrict_outputs, pod.py:95-97), the
 * interface decoder -- WFPC: the full map (driver.py:398-402); SRPC: its
 * restriction to the `gio` outputs (driver.py:400-402), gio then indexes
 * that restriction (0..n_gio-1) --, the sampled residual rows and the local
 * column order of RestrictedResidual (driver.py:392-396,
 * partition.py:361-425), the constraint matrix, and for gappy HR the
 * weights pinv(basis[rows]) (hyper.py:153-160). */
typedef struct {
  int32_t n_int, n_gam;      /* latent dims of this block */
  ddnm_decoder interior;     /* n_out == n_io */
  ddnm_decoder interface;    /* WFPC: n_out == N_Gamma; SRPC: n_out == n_gio */
  int32_t n_rows;            /* HR sample rows */
  const int64_t* res_rows;   /* [n_rows] global residual rows, sorted */
  int32_t n_cols;            /* n_io + n_gio */
  const int64_t* cols;       /* [n_cols] global state columns, local order */
  int32_t n_io;
  int32_t n_gio;
  const int64_t* gio;        /* [n_gio] positions in the interface outputs */
  const double* CA;          /* WFPC: C @ A_i [n_c][N_Gamma] (driver.py:368-369);
                                SRPC: Ahat_i [n_c][n_gam] (driver.py:375) */
  int32_t n_basis;           /* gappy HR: residual basis size; 0 = collocation */
  const double* weights;     /* gappy HR: [n_basis][n_rows] */
} ddnm_block;

/* Thin-plate-spline RBF initializer (driver.py:59-90 + scipy RBFInterpolator
 * evaluation): x0 = [phi(|qn*eps - y_i*eps|)_i, prod(((qn-shift)/scale)^p_r)_r]
 * @ coeffs with qn = (mu - lo)/span. */
typedef struct {
  int32_t n_centers, n_mono;
  const double* y;           /* [n_centers][2] */
  const double* coeffs;      /* [n_centers + n_mono][n_D] */
  const int64_t* powers;     /* [n_mono][2] */
  double shift[2], scale[2], lo[2], hi[2];
  double epsilon;
} ddnm_rbf;

typedef struct {
  int32_t abi_version;       /* DDNM_ABI_VERSION */
  int32_t map_kind;          /* DDNM_MAP_* (same for every block) */
  int32_t activation;        /* DDNM_ACT_* of the interior maps */
  int32_t gam_activation;    /* DDNM_ACT_* of the interface maps (SRPC port nets: sigmoid) */
  int32_t constraint_mode;   /* DDNM_CON_* */
  int32_t nx, ny;            /* interior FD grid (burgers.py:67-106) */
  double nu;
  int32_t n_blocks;
  int32_t n_c;               /* multipliers (WFPC test-matrix rows) */
  const ddnm_block* blocks;  /* [n_blocks] */
  ddnm_rbf rbf;              /* n_centers == 0: no initializer */
} ddnm_artifacts;

/* SqpConfig (sqp.py:68-81) */
typedef struct {
  double tol;
  int32_t max_iter;
  double armijo_c1;
  double backtrack_factor;
  int32_t max_halvings;
  double reg_scale;
} ddnm_sqp_cfg;

typedef struct {
  int32_t n_primal;          /* n_D = sum (n_int + n_gam) */
  int32_t n_mult;            /* n_C */
  int32_t n_blocks;
  int32_t total_rows;        /* sum of HR sample rows over blocks */
  int32_t total_out_rows;    /* sum of HR output rows (gappy: n_basis, else n_rows) */
  int32_t total_out_R;       /* sum of out rows * (n_int + n_gam) */
  int32_t total_int_out;     /* sum n_io */
  int32_t total_gam_out;     /* sum N_Gamma */
  int32_t total_R;           /* sum n_rows * (n_int + n_gam) */
  int32_t total_cjac;        /* sum n_c * n_gam */
  int32_t total_int_J;       /* sum n_io * n_int */
  int32_t total_gam_J;       /* sum N_Gamma * n_gam */
  int32_t slots_per_cta;     /* mu processed concurrently per CTA */
  int32_t ctas;              /* persistent grid size */
  int32_t smem_bytes;        /* dynamic shared memory per CTA */
  int32_t device;
  int32_t eval_units;        /* evaluation units the blocks are split into (0: whole
                                blocks); blocks too large for one CTA (configs 3/4)
                                are evaluated as chunks of their sampled rows plus
                                chunks of interface outputs; DDNM_UNIT_ROWS=<rows>
                                forces the split (tests) */
  int32_t wide;              /* 1: the batch-wide engine (one lane per mu, csrc/ddnm_wide.h)
                                is available for this instance */
} ddnm_info;

/* Per-mu solve results; every pointer may be NULL except x and lam. */
typedef struct {
  double* x;                 /* [B][n_D]   SqpResult.x   (best iterate on line-search failure) */
  double* lam;               /* [B][n_C]   SqpResult.lam */
  int32_t* n_iter;           /* [B] accepted steps */
  int32_t* n_evals;          /* [B] eval_gradients calls inside iterate */
  int32_t* status;           /* [B] DDNM_STATUS_* */
  int32_t* n_reg;            /* [B] regularized KKT solves (RuntimeWarning count) */
  double* merit;             /* [B] merit_history[-1] */
  double* objective;         /* [B] objective_history[-1] */
  double* merit_hist;        /* [B][max_iter+1], NaN padded */
  double* obj_hist;          /* [B][max_iter+1], NaN padded */
  double* alpha_hist;        /* [B][max_iter],   NaN padded */
  double* x0;                /* [B][n_D] initial latents used */
  double* lam0;              /* [B][n_C] initial multipliers used */
} ddnm_solve_out;

/* One eval_gradients (sqp.py:117-146) per mu at a given (x, lam), with every
 * intermediate of the HR closure (driver.py:404-432) for parity tests.
 * Per-block arrays are concatenated over blocks in block order.  Any pointer
 * may be NULL. */
typedef struct {
  double* rho;               /* [B][n_D] */
  double* con;               /* [B][n_C] */
  double* merit;             /* [B] */
  double* objective;         /* [B] */
  double* Br;                /* [B][total_out_rows] (the weighted rows for gappy HR) */
  double* R;                 /* [B][total_out_R] per block [out rows][n_int+n_gam] = [R_int | R_gam] */
  double* cval;              /* [B][n_blocks][n_C] */
  double* cjac;              /* [B][total_cjac] per block [n_C][n_gam] */
  double* int_g;             /* [B][total_int_out] interior subnet outputs */
  double* int_J;             /* [B][total_int_J] */
  double* gam_g;             /* [B][total_gam_out] interface decoder (WFPC: full) */
  double* gam_J;             /* [B][total_gam_J] */
  double* bvals;             /* [B][total_rows][3] sampled (bx, by, c) of assemble() */
  double* step;              /* [B][n_D + n_C] KKT step (s, s_lam) at (x, lam) */
  int32_t* kkt_status;       /* [B] 0 ok, 1 regularized, 2 singular */
} ddnm_eval_out;

typedef struct ddnm_ctx ddnm_ctx;

/* Host-only (no GPU): the evaluation units ddnm_ctx_create would split these
 * artifacts into (0 when every block is evaluated whole).  row_unit
 * [total_rows] (nullable): the unit of every sampled row, block by block;
 * unit_info [n_units][8] (nullable; size it by a first call with both NULL):
 * real block, UF_* flags (1 rows, 2 constraint, 4/8 accumulate), rows,
 * interior outputs, interior hidden units, interface outputs, interface
 * hidden units, constraint columns. */
int ddnm_plan_units(const ddnm_artifacts* art, int32_t* n_units, int32_t* row_unit,
                    int32_t* unit_info);

/* Host-only (no GPU): how the batch-wide engine (csrc/ddnm_wide.h) would lay
 * these artifacts out.  info10: [0] eligible (else ddnm_last_error says why
 * not), [1] sweep tiles, [2] coarse and [3] fine decoder parts, [4] row
 * chunks, [5] constraint chunks, [6] W2 stream slots (tile steps x outputs per
 * tile), [7] stored decoder entries (their ratio is the sweep's useful
 * fraction), [8] g / J doubles per lane, [9] longest window union of a tile
 * (<= 32, the hidden ring).  tile_of_output (nullable): the tile of every
 * decoder output, concatenated block by block (interior, then interface). */
int ddnm_wide_plan(const ddnm_artifacts* art, int32_t* info10, int32_t* tile_of_output);

const char* ddnm_last_error(void);
int ddnm_abi_version(void);

/* Upload the artifacts and plan the kernels.  device < 0 selects the current
 * device.  slots_per_cta <= 0 picks the default for the instance. */
int ddnm_ctx_create(int32_t device, const ddnm_artifacts* art,
                    int32_t slots_per_cta, ddnm_ctx** out);
int ddnm_ctx_destroy(ddnm_ctx* ctx);
int ddnm_ctx_info(const ddnm_ctx* ctx, ddnm_info* info);

/* Batched solve_rom (driver.py:554-597, compute_error=False) for B parameters
 * mu[B][2] = (a, lambda).  x0 == NULL: RBF initial latents on device
 * (driver.py:82-90); lam0 == NULL: least-squares multipliers on device
 * (driver.py:461-471).  Host pointers; copies are synchronous. */
int ddnm_solve_batch(ddnm_ctx* ctx, int32_t B, const double* mu,
                     const double* x0, const double* lam0,
                     const ddnm_sqp_cfg* cfg, ddnm_solve_out* out);

/* Same with device-resident inputs/outputs, on `stream` (a cudaStream_t;
 * NULL = the context's stream).  The slot engine is one asynchronous launch;
 * the wide engine (ddnm_ctx_set_engine below) enqueues its SQP rounds on the
 * stream, reads the running count every few rounds, and returns when the batch
 * is solved. */
int ddnm_solve_batch_device(ddnm_ctx* ctx, int32_t B, const double* d_mu,
                            const double* d_x0, const double* d_lam0,
                            const ddnm_sqp_cfg* cfg, ddnm_solve_out* d_out,
                            void* stream);

/* Batched eval_gradients at (x, lam) with all intermediates (host pointers). */
int ddnm_eval_batch(ddnm_ctx* ctx, int32_t B, const double* mu,
                    const double* x, const double* lam, double reg_scale,
                    ddnm_eval_out* out);

/* Device work counters of the last solve (for the roofline): total block
 * evaluations and KKT solves executed. */
int ddnm_last_counters(const ddnm_ctx* ctx, int64_t* evals, int64_t* kkts);

/* Which engine ddnm_solve_batch[_device] runs: the persistent kernel (one CTA
 * slot per mu, the whole SQP loop in one launch) or the batch-wide engine (one
 * lane per mu, rounds of evaluation + SQP-step kernels looped inside the
 * library; available when ddnm_info.wide: autoencoder maps, WFPC coupling,
 * collocation HR, banded decoders).  AUTO (default): wide when available
 * (environment: DDNM_WIDE=0/1 forces, DDNM_WIDE_MIN_B=<batch> sets the
 * smallest batch that goes wide).  Both engines take the same decisions on the
 * same evaluations (sqp.py:230-299); their evaluations differ by rounding. */
#define DDNM_ENGINE_AUTO 0
#define DDNM_ENGINE_SLOTS 1
#define DDNM_ENGINE_WIDE 2
int ddnm_ctx_set_engine(ddnm_ctx* ctx, int32_t engine);
/* SQP rounds and kernel launches of the last batched solve (slots: 0 and 1). */
int ddnm_last_rounds(const ddnm_ctx* ctx, int64_t* rounds, int64_t* launches);
/* Evaluations (lanes) the wide engine launched in the last solve, including
 * speculative candidates that were not consumed (ddnm_last_counters counts
 * the consumed ones). */
int ddnm_last_lanes(const ddnm_ctx* ctx, int64_t* lanes);

/* Device-side phase profile of the last solve when the environment variable
 * DDNM_PROF is set (SM clock cycles summed over CTAs, thread 0 of each CTA):
 * [0] slot fetch, [1..4] eval phases A-D, [5] slot init, [6] SQP state
 * machine, [7] KKT, [8..15] reserved.  All zero when profiling is off. */
int ddnm_last_profile(const ddnm_ctx* ctx, uint64_t* cycles16);

/* ---- full decode (RomInstance.decode, driver.py:148-152) ---------------- */

/* Register the full maps: interior[b] is block b's whole interior decoder
 * (n_out = all interior dofs; the ddnm_block carries only its HR
 * restriction), same latent dim, map kind and activation as the artifacts.
 * interface[b] is its whole interface decoder; NULL (WFPC only) uses the
 * blocks' `interface` decoders, which are already whole. */
int ddnm_ctx_set_full_decoders(ddnm_ctx* ctx, const ddnm_decoder* interior,
                               const ddnm_decoder* interface);

/* Length of one decoded state: sum over blocks of (interior n_out + N_Gamma),
 * laid out [blk0 interior | blk0 interface | blk1 interior | ...] -- the
 * flattened list of (x_int, x_gam) pairs RomInstance.decode returns. */
int ddnm_ctx_state_len(const ddnm_ctx* ctx, int64_t* len);

/* Decode B latent solutions x[B][n_D] into states[B][state_len] (NULL: not
 * stored).  fom (NULL allowed) holds restrict_blocks (driver.py:477-480) of a
 * FOM state per mu in the same layout; then err[B] = relative_error
 * (driver.py:496-507), NaN where a reference block has zero norm (the
 * reference raises ValueError there).  fom and err are both NULL or both set.
 * Host pointers, synchronous. */
int ddnm_decode_batch(ddnm_ctx* ctx, int32_t B, const double* x,
                      const double* fom, double* states, double* err);

/* Same with device pointers, asynchronous on `stream` (NULL: context stream). */
int ddnm_decode_batch_device(ddnm_ctx* ctx, int32_t B, const double* d_x,
                             const double* d_fom, double* d_states,
                             double* d_err, void* stream);


/* ---- subdomain-sharded solve -------------------
 * Round-synchronous batched SQP in which each rank evaluates only its blocks
 * [blk_lo, blk_hi) of every mu (the HR residual closures of driver.py:404-432
 * and the constraint closures, one SqpBlock each, sqp.py:28-41), the block
 * pieces (Gram H_b = R_b^T R_b, R_b^T r_b, cval_b, cjac_b, r_b^T r_b -- what
 * eval_gradients and _kkt_matrix need of a block, sqp.py:117-159) are
 * all-gathered, and every rank then runs the identical SQP decision and KKT
 * solve (sqp.py:230-299), so all ranks hold bit-identical results.  The
 * caller owns the collective (NCCL all-gather between the eval and the step);
 * with one rank the packets are the gathered buffer.  Device pointers; all
 * work is asynchronous on `stream` -- the caller's cudaStream_t, used as is
 * (0 is the legacy default stream, not the context's stream), so kernels
 * order with the caller's collective -- except where a count is returned. */
typedef struct ddnm_dd ddnm_dd;

/* Doubles of one mu's packet for blocks [blk_lo, blk_hi). */
int ddnm_dd_packet_len(const ddnm_ctx* ctx, int32_t blk_lo, int32_t blk_hi, int64_t* len);

/* Start a sharded solve of B parameters (device arrays as in
 * ddnm_solve_batch_device); this rank evaluates blocks [blk_lo, blk_hi).
 * Results are written to d_out as slots finish.  n_active (host, may be
 * NULL) receives the number of running mu (synchronises the stream). */
int ddnm_dd_begin(ddnm_ctx* ctx, int32_t B, const double* d_mu, const double* d_x0,
                  const double* d_lam0, const ddnm_sqp_cfg* cfg, int32_t blk_lo,
                  int32_t blk_hi, const ddnm_solve_out* d_out, void* stream,
                  ddnm_dd** out, int32_t* n_active);

/* This rank's block pieces at every running mu's trial point:
 * d_packets[B][pk_stride] (pk_stride >= ddnm_dd_packet_len of the range). */
int ddnm_dd_eval(ddnm_dd* dd, double* d_packets, int64_t pk_stride, void* stream);

/* One SQP round from the gathered pieces d_gathered[nranks][B][pk_stride];
 * rank r evaluated blocks [bounds[r], bounds[r+1]) (bounds[0] = 0,
 * bounds[nranks] = n_blocks).  n_active as in ddnm_dd_begin. */
int ddnm_dd_step(ddnm_dd* dd, const double* d_gathered, int32_t nranks,
                 const int32_t* bounds, int64_t pk_stride, void* stream,
                 int32_t* n_active);

/* ddnm_dd_eval with the all-gather fused in: the kernel stores this rank's
 * packets straight into every rank's gathered buffer, at
 * peers[r] + (rank * B + mu) * pk_stride, over NVLink (peer stores; peers[r]
 * valid on this device: same-process peer access or ddnm_ipc_open_handle).
 * Protocol: every rank owns TWO gathered buffers and round t uses buffer
 * t % 2 on all ranks; after ddnm_dd_eval_p2p of round t, a cross-rank barrier
 * ordered on `stream` (e.g. a one-element NCCL all-reduce), then
 * ddnm_dd_step on this rank's buffer t % 2.  A faster peer's stores of round
 * t + 1 go to the other buffer, and the barrier of round t + 1 orders every
 * rank's step t before any store of round t + 2 into buffer t % 2.  With one
 * buffer the protocol is racy: a peer's round-(t+1) stores could overwrite
 * packets this rank's step t is still reading. */
int ddnm_dd_eval_p2p(ddnm_dd* dd, double* const* peers, int32_t nranks, int32_t rank,
                     int64_t pk_stride, void* stream);

/* Trial records: per mu [running flag, x_trial[n_D]] (+ padding), the input
 * of the next ddnm_dd_eval.  By default the handle owns them (B records) and
 * ddnm_dd_step advances every mu.  Sharding the steps by mu (each mu solved
 * by one rank; the KKT work divides by the rank count): every rank gives a
 * buffer of cap >= B records, the same slice size on every rank, and its mu
 * slice [mu_lo, mu_hi); ddnm_dd_step then advances only that slice and writes
 * its records, and the caller all-gathers the records (rank-major chunks of
 * cap / nranks records) before the next ddnm_dd_eval; n_active counts the
 * slice (sum it over the ranks).  The final results are written by the
 * owning rank only: gather the slices' rows. */
int ddnm_dd_trial_len(const ddnm_dd* dd, int64_t* len);
int ddnm_dd_set_trials(ddnm_dd* dd, double* d_trials, int64_t cap, int32_t mu_lo,
                       int32_t mu_hi, void* stream);

int ddnm_dd_end(ddnm_dd* dd);

/* Evaluate with the batch-wide kernels (one lane per mu; csrc/ddnm_wide.h)
 * instead of one CTA slot per mu: for a handle that owns every block
 * (blk_lo = 0, blk_hi = n_blocks) of an eligible instance (autoencoder maps,
 * WFPC coupling, collocation HR, banded decoders).  ddnm_dd_eval then writes
 * one packet per LANE (a running mu may come with several candidate step
 * lengths per round), so d_packets must hold max(2 * roundup32(B), 1024) rows;
 * ddnm_dd_step reads them from the same buffer with nranks = 1.
 * on = 2: one candidate per mu and packets [B][pk_stride] exactly as
 * ddnm_dd_eval lays them out, for any block range -- the evaluation of a rank
 * of a subdomain-sharded solve (the all-gather and ddnm_dd_step are unchanged;
 * not with ddnm_dd_eval_p2p).  ddnm_solve_batch[_device] takes this path by
 * itself for large batches (DDNM_WIDE=0/1 forces). */
int ddnm_dd_set_wide(ddnm_dd* dd, int32_t on);

/* CUDA IPC of a device buffer between the processes of one node (64-byte
 * handles, exchanged by the caller), for ddnm_dd_eval_p2p's peer buffers.
 * A handle maps the start of the cudaMalloc allocation holding dptr, so the
 * exported buffer must be a whole allocation: ddnm_dev_alloc (zeroed). */
int ddnm_dev_alloc(int32_t device, int64_t bytes, void** out);
int ddnm_dev_free(void* p);
int ddnm_ipc_get_handle(const void* dptr, unsigned char* handle);
int ddnm_ipc_open_handle(const unsigned char* handle, void** dptr);
int ddnm_ipc_close_handle(void* dptr);


/* ---- binio (binio.py:1-87) and instance files -------------------------------
 * The reference's language-neutral matrix format: magic "DDNMROM1", then per
 * record u32 name length, UTF-8 name, u64 rows, u64 cols, rows*cols float64
 * in column-major order, all little-endian (binio.py:1-8).  Reading checks
 * the magic, truncation and overruns as read_matrices does (binio.py:43-70);
 * writing is byte-identical to write_matrices (binio.py:22-40). */
typedef struct ddnm_binio ddnm_binio;

int ddnm_binio_read(const char* path, ddnm_binio** out);
int ddnm_binio_count(const ddnm_binio* b, int64_t* n);
/* Record i: name bytes and their length (valid until ddnm_binio_free; a
 * name may contain NUL bytes), shape, column-major data. */
int ddnm_binio_entry(const ddnm_binio* b, int64_t i, const char** name, int64_t* name_len,
                     int64_t* rows, int64_t* cols, const double** data);
/* Record by name (the last one if repeated, as the reference's dict). */
int ddnm_binio_find(const ddnm_binio* b, const char* name, int64_t* rows, int64_t* cols,
                    const double** data);
int ddnm_binio_free(ddnm_binio* b);
/* n records; data[k] column-major [rows[k] x cols[k]]; name_lens NULL:
 * NUL-terminated names. */
int ddnm_binio_write(const char* path, int64_t n, const char* const* names,
                     const int64_t* name_lens, const int64_t* rows, const int64_t* cols,
                     const double* const* data);

/* A context straight from an instance file pair: `path` (binio, every
 * artifact array of ddnm_artifacts as a record named as in the package's
 * .npz artifacts, integer arrays stored as float64 like the reference stores
 * CSR indices, save_net autoencoder.py:424-450) and the meta file next to it
 * (same stem, ".txt", binio.py:73-87 format, "format = ddnm-instance-1").
 * Also registers the full decoders when the file has them.  No Python. */
int ddnm_ctx_create_binio(int32_t device, const char* path, int32_t slots, ddnm_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* DDNM_H */
