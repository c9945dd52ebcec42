// Device side of the batched DD NM-ROM-HR online solve (sm_100a, FP64).
//
// One persistent CTA owns G "slots"; each slot runs one parameter mu through
// the reference's whole online solve (driver.solve_rom, driver.py:554-597):
// boundary data (burgers.py:188-210), RBF initial guess (driver.py:82-90),
// least-squares multipliers (driver.py:461-471) and the Lagrange-Gauss-Newton
// SQP loop (sqp.py:230-299).  All slots of a CTA advance in lock-step
// "rounds": every round evaluates one trial point per active slot
// (eval_gradients, sqp.py:117-146) and then advances each slot's state
// machine (Armijo test, KKT solve, bookkeeping).  A finished slot pulls the
// next mu from a global work counter, so line-search divergence between
// parameters never idles a CTA (the batch is load-balanced at mu granularity).
//
// Per block the round is four CTA-wide phases separated by __syncthreads:
//   A  hidden units of the interior subnet and the interface decoder:
//      z = b1 + sum_d W1[:,d] x_d (latent-column order, hyper.py:184-188),
//      swish(z), swish'(z) (autoencoder.py:31-45)           -> smem
//   B  CSR output sweep, g and J together (hyper.py:190-197) -> smem
//   C  WFPC constraint CA g, CA J (driver.py:371-373) and the HR stencil
//      residual + dense Jacobian row + chain rule (partition.py:427-464,
//      driver.py:422-429)                                    -> smem
//   D  Gram block H = R^T R, R^T r and r^T r (sqp.py:137-139,155) -> slot buffer
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ddnm {

constexpr int MAXB = 16;        // subdomain blocks
constexpr int MAXE = 6;         // stencil entries per residual row
constexpr int WARP = 32;

enum MapKind { MAP_AE = 0, MAP_LINEAR = 1 };
enum Act { ACT_SWISH = 0, ACT_SIGMOID = 1 };
enum Phase { PH_IDLE = 0, PH_INIT = 1, PH_TRIAL = 2, PH_DONE = 3 };
enum Status { ST_OK = 0, ST_LINE_SEARCH = 1, ST_KKT_SINGULAR = 2, ST_LSTSQ_RANK = 3 };

struct DecDev {
  int n_out, n_hidden;
  int act;                // ACT_* of this map (SRPC port nets are Sigmoid)
  const double* W1;       // LINEAR: Phi [n_out][lat]  (AE: unused on device)
  const double* W1t;      // AE: W1 transposed [lat][ldw] (coalesced per latent column),
  int ldw;                //     ldw = n_hidden + 32, zero padded
  const double* b1;       // [n_hidden]
  const int* indptr;      // [n_out+1]
  const int* indices;     // [nnz]
  const double* data;     // [nnz]
  const double* scale;    // [n_out]
  const double* shift;    // [n_out]
  int ell_w;              // ELL width (max nnz per row, padded to 8)
  const double* ell_v;    // [ell_w][n_out] W2 values in storage order, 0-padded
  const double* ell_zero; // 1 zero double (target of masked-out lanes)
  const int* ell_k;       // [ell_w][n_out] hidden indices, 0-padded (null if contiguous)
  const int* ell_k0;      // [n_out] first hidden index when every row's window is contiguous
  // DMMA sweep (contiguous windows only): W1 in mma.m8n8k4 A-fragment order,
  // W2 rows contiguous, and tiles of consecutive outputs with their k-block range
  const double* w1frag;   // [ceil(n_hidden/4)][32]: lane -> W1[4kb + (lane&3)][lane>>2]
  const double* v_row;    // [n_out][ell_w] W2 values, row-contiguous, 0-padded
  const int* row_w;       // [n_out] stored entries per row
  // chained tensor-core sweep: W1 as the B operand, [ceil(n_hidden/4)][32]:
  // lane -> k = 4kb + (lane&3), n = lane>>2: W1[k][n] (n < lat), 1 (n == lat), 0
  const double* wbfrag;
  // hidden pre-activation on the FP64 tensor cores (hidden_group): W1 as the
  // m8n8k4 A operand, [ceil(n_hidden/8)][ceil(lat/4)][32]:
  // lane -> W1[8t + (lane>>2)][4ks + (lane&3)] (0 outside)
  const double* w1a;
};

// Chained tensor-core sweep (sweep_chain): a tile is 8 consecutive outputs of
// one decoder with its k-block range [lo, hi] and the offset of its A
// fragments (the banded W2 block, one 32-double fragment per k-block); a
// chain is a run of consecutive tiles one warp walks k-block by k-block.
// The host also flattens each chain's walk into steps: the k-block, the A
// fragment index of each ring slot's live tile (-1: none) and the slots whose
// tile ends there, so the device loop prefetches the next step's fragments.
struct TileV2 { int o0, cnt, lo, hi, aoff; };
struct ChainRec { int which, t0, nt, s0, ns; };     // which: 0 interior, 1 interface
struct StepRec { int kb, last; int aidx[4]; };

// A tensor-core sweep tile: up to 8/G consecutive outputs of one decoder with
// everything its B operand needs, so a warp issues no dependent loads.
struct TileRec {
  int o0, cnt, kb_lo, kb_hi;    // cnt | which << 8 (0 interior, 1 interface)
  int k0[8];                    // first hidden unit of each output's window
  int w[8];                     // stored entries of each output
};

// Sampled residual rows in local-column form (RestrictedResidual,
// partition.py:372-425), structure of arrays so consecutive rows (lanes) read
// consecutive addresses.  Entry e of row r is at [e * n_rows + r]; entries are
// sorted by global column, the storage order of the reference's Bx/By/Cdiff
// rows, so the per-operator sums accumulate in the reference order.
struct StRows {
  const int* gu;          // local position of u_p
  const int* gv;          // local position of v_p
  const int* nent;        // distinct local columns referenced (<= 6)
  const int* bflags;      // bit0 left, bit1 right, bit2 bottom, bit3 top, bit4 v-row
  const int* col;         // [MAXE][n_rows] local columns
  const int* src;         // [MAXE][n_rows] source codes: >= 0 interior output, < 0: -1 - interface output
  const int* src_gu;      // source codes of u_p and v_p
  const int* src_gv;
  const double* bxc;      // [MAXE][n_rows]
  const double* byc;
  const double* cdc;
  const double* xc;       // node coordinates (ghost points share one of them)
  const double* yc;
};

struct BlockDev {
  // (tiles depend on G; the host builds them for the kernel's G)
  int ni, ng, w;          // latent dims, w = ni + ng
  int nrows, n_io, n_gio;
  int xoff;               // offset of (x_int, x_gam) in the stacked latent
  int row_off;            // offset in concatenated rows (bvals, Br)
  int iout_off, gout_off, R_off, cjac_off, intJ_off, gamJ_off;
  int eb_off;             // offset of this block inside a slot eval buffer
  DecDev in, ga;
  const TileRec* tiles;   // tensor-core sweep tiles of both decoders (or null)
  int n_tiles, n_tiles_in;  // total, interior (stored first)
  const double* tile_v;   // [n_tiles][10][32] B-operand W2 values per tile
  const TileV2* t2;       // chained sweep tiles (interior, then interface)
  const double* afr;      // their A fragments
  const ChainRec* chains; // chains of tiles (null: per-output sweep)
  const StepRec* steps;   // their k-block walks
  int n_chains;
  int chain_gam_only;     // 1: chains cover the interface decoder only (the
                          //    interior runs the per-output sweep)
  StRows rows;
  const int* gio;
  const double* CA;       // WFPC: C A_i [n_c][ga.n_out]; SRPC: Ahat_i [n_c][ng]
  int nbz;                // gappy HR: residual basis size (0: collocation)
  const double* wts;      // gappy HR: weights [nbz][nrows] (hyper.py:153-160)
  int out_off, outR_off;  // offsets of the weighted rows in the Br / R dumps
  // evaluation units (large blocks split into row chunks, see Params::units):
  int uflags;             // UF_* below
  int real;               // real block of this unit
  const int* iout_map;    // [in.n_out] real-block interior output of each unit output (null: identity)
  const int* gout_map;    // [ga.n_out] real-block interface output (null: identity)
  const int* row_map;     // [nrows] real-block row of each unit row (null: identity)
};

// evaluation-unit flags: a unit with rows evaluates its stencil rows and adds
// its Gram contribution to its real block; a constraint unit evaluates
// C A_i g over its interface outputs.  ACC_*: add into the real block's
// pieces (a later unit of the same block) instead of writing them.
enum UnitFlags { UF_ROWS = 1, UF_CON = 2, UF_ACC_GRAM = 4, UF_ACC_CON = 8 };

struct SlotState {
  int mu, phase, n_iter, n_trials, n_evals, n_reg, status, need_kkt;
  int lam_given, pad;
  double alpha, merit, obj, best_merit;
};

struct SqpCfg {
  double tol, c1, factor, reg_scale;
  int max_iter, max_halvings;
};

struct SolveOut {
  double *x, *lam, *merit, *objective, *merit_hist, *obj_hist, *alpha_hist, *x0, *lam0;
  int *n_iter, *n_evals, *status, *n_reg;
};

struct EvalOut {
  double *rho, *con, *merit, *objective, *Br, *R, *cval, *cjac, *int_g, *int_J,
      *gam_g, *gam_J, *bvals, *step;
  int* kkt_status;
};

struct Params {
  int nb, n_D, n_C, nK, map_kind, act;
  int con_mode;           // 0 WFPC (CA g^Gamma), 1 SRPC (Ahat x_Gamma)
  int nx, ny;
  double nu, hx, hy;
  int total_rows;
  int tot_iout, tot_intJ, tot_gout, tot_gamJ, tot_R, tot_cjac;
  BlockDev blk[MAXB];
  // RBF initializer
  int rbf_P, rbf_R;
  const double* rbf_y;
  const double* rbf_coeffs;
  const int* rbf_pow;
  double rbf_shift[2], rbf_scale[2], rbf_lo[2], rbf_hi[2], rbf_eps;
  // shared-memory plan (offsets in doubles from the dynamic smem base)
  int G;                  // slots per CTA (== template G)
  int sm_state;           // SlotState[G]
  int sm_vec;             // per slot: x, lam, s, slam, xt, lt, bx, bl, rho_t (nK each)
  int sm_eb;              // per slot: 2 eval buffers of eb_size
  int eb_size;
  int eb_rho, eb_con, eb_scal;  // inside an eval buffer: rho[n_D], con[n_C], (merit, obj)
  int sm_scr;             // per slot scratch (scr_size)
  int scr_size;
  int scr_sig, scr_dsig, scr_gint, scr_jint, scr_ggam, scr_jgam, scr_R, scr_r;
  int scr_RB;             // gappy: weighted [R | r] rows [max nbz][W + 1], or -1
  int tot_out, tot_outR;  // sum over blocks of HR output rows (nbz or nrows), x W
  int nh_tot;             // max over blocks of (int hidden + gam hidden)
  // work
  int B;
  const double* mu;       // [B][2]
  const double* x0_in;    // [B][n_D] or null
  const double* lam0_in;  // [B][n_C] or null
  SqpCfg cfg;
  SolveOut so;
  EvalOut eo;
  int eval_mode;          // 1: single eval with dumps (ddnm_eval_batch)
  int eval_step;          // eval mode: also solve the KKT
  double* gbv;            // per global slot [total_rows][3] boundary values
  double* gJ;             // per global slot interior-decoder Jacobian rows [n_io][n_int]
  int gJ_stride;
  double* gJg;            // per global slot interface-decoder Jacobian rows [N_gam][n_gam]
  int gJg_stride;
  int* work;              // [0]: next mu; [1]: finished CTAs
  unsigned long long* counters;  // [0] block-evals, [1] KKT solves
  unsigned long long* prof;      // [15] per-phase clock totals (DDNM_PROF=1), or null
  // blocks evaluated by eval_blocks: [b_lo, b_hi) (all blocks except in k_dd_eval)
  int b_lo, b_hi;
  // round-synchronous subdomain-sharded solve (k_dd_eval / k_dd_step)
  SlotState* dd_st;       // [B] per-mu SQP state
  double* dd_vec;         // [B][8][nK] x, lam, s, slam, xt, lt, best x, best lam
  double* dd_ecur;        // [B][eb_size] current (accepted) evaluation
  double* dd_pk;          // [B][pk_stride] this rank's block pieces (k_dd_eval)
  const double* dd_gath;  // [dd_nranks][B][pk_stride] gathered pieces (k_dd_step)
  int pk_stride, dd_nranks, dd_init;
  int dd_bnd[MAXB + 1];   // block range of rank r: [dd_bnd[r], dd_bnd[r+1])
  int* dd_active;         // k_dd_step: count of slots still running
  // trial records [mu][dd_rec]: running flag, then the trial point x_t (the
  // next evaluation's input on every rank); k_dd_step writes the records of
  // the mu it advances, [dd_mu_lo, dd_mu_hi) (its slice), k_dd_eval reads all
  double* dd_trial;
  int dd_rec, dd_mu_lo, dd_mu_hi;
  // batch-wide evaluation (ddnm_wide.cu): dd_gath holds one packet per lane;
  // mu's candidates are rows dd_vbase[mu] .. + dd_kof[mu] - 1 (null: one
  // packet per mu per rank, the subdomain-sharded layout above)
  const int* dd_vbase;
  const int* dd_kof;
  // dense-fallback KKT workspace per global slot (null: the slot's own scratch)
  double* kkt_fb;
  long long kkt_fb_stride;
  // peer-memory all-gather fused into k_dd_eval: when dd_npeers > 0 the
  // packets go straight to every rank's gathered buffer (NVLink stores)
  double* dd_peers[MAXB];
  int dd_npeers, dd_rank;
  // largest block system (W + n_C) the block-structured KKT is tried on
  // (<= 96); larger ones go straight to the dense LU
  int kkt_block_max;
  // hidden layer: 1 = FP64 tensor-core tiles (hidden_group), 0 = per-unit DFMA
  int hid_dmma;
  // KKT workspace in global memory (kernels instantiated with KG = true)
  double* kkt_g;          // per global slot [kkt_stride]
  long long kkt_stride;
  // the two evaluation buffers of every slot in global memory (L2) instead of
  // shared memory, [global slot][2][eb_size] (null: shared memory); chosen by
  // the planner when they would cost slots (config 4: 16 blocks x 345
  // doubles x 2 per slot)
  double* eb_glob;
  // evaluation units: when non-null, eval_blocks walks units[u_bnd[b]] ..
  // units[u_bnd[b + 1] - 1] for real block b instead of blk[b] (blocks too
  // large for one CTA's shared memory are split into chunks of their sampled
  // rows, each with the decoder subnet restricted to the outputs its rows
  // reference, plus chunks of interface outputs for the WFPC constraint)
  const BlockDev* units;
  int n_units;
  int u_bnd[MAXB + 1];
};

// RomInstance.decode (driver.py:148-152): one full decoder of one block.
struct DecodeJob {
  DecDev D;               // full interior map (job 2b) or the interface map (2b+1)
  int x_off, lat;         // latent slice of the stacked x
  int out_off;            // offset in the flattened per-mu state
};

struct DecodeParams {
  const DecodeJob* jobs;  // [n_jobs] (device)
  int n_jobs, nb, B, n_D, state_len, act, linear, mu_tile, max_hidden;
  const double* x;        // [B][n_D]
  const double* fom;      // [B][state_len] restrict_blocks of a FOM state, or null
  double* states;         // [B][state_len] or null
  double* part;           // [B][n_jobs][2] (sum (f-r)^2, sum f^2) when fom
  double* err;            // [B] relative_error (driver.py:496-507) when fom
};


// ---------------------------------------------------------------------------
// scalar helpers

// 2^(j/32), j = 0..31 (correctly rounded)
static __device__ const double k_exp2_32[32] = {
    0x1.0000000000000p+0, 0x1.059b0d3158574p+0, 0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, 0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0,
    0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123422p+0, 0x1.44e086061892dp+0,
    0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
    0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0,
    0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0};

// exp(x) for |x| <= 700: x = (32 m + j) ln2/32 + r, |r| <= ln2/64,
// exp(x) = 2^m 2^(j/32) (1 + p(r)), p degree 6 (truncation < 4e-18).
// 11 FP64 ops + integer exponent arithmetic (vs ~23 for the libdevice exp).
__device__ __forceinline__ double exp_fast(double x, const double* tab) {
  const double t = fma(x, 0x1.71547652b82fep+5, 6755399441055744.0);  // 32/ln2, 1.5*2^52
  const int n = __double2loint(t);
  const double nd = t - 6755399441055744.0;
  double r = fma(nd, -0x1.62e42fee00000p-6, x);                       // ln2/32 (hi, 32 bits)
  r = fma(nd, -0x1.a39ef35793c76p-38, r);                             // ln2/32 (lo)
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = p * r;                                                          // exp(r) - 1
  const double T = __ldg(tab + (n & 31));
  const double y = fma(T, p, T);
  return __hiloint2double(__double2hiint(y) + ((n >> 5) << 20), __double2loint(y));
}

__device__ __forceinline__ double rcp_fast(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

// scipy.special.expit(z) = 1 / (1 + exp(-z)); |z| clamped at 700 (the
// results are exactly 1 or below 1e-304 there anyway)
__device__ __forceinline__ double expit_fast(double z, const double* tab) {
  const double x = fmin(fmax(-z, -700.0), 700.0);
  return rcp_fast(1.0 + exp_fast(x, tab));
}

__device__ __forceinline__ void act_pair(int act, double z, double& a, double& da, const double* tab) {
  const double s = expit_fast(z, tab);
  if (act == ACT_SWISH) {
    a = z * s;                                   // autoencoder.py:33
    da = s * fma(z, 1.0 - s, 1.0);               // autoencoder.py:42
  } else {
    a = s;
    da = s * (1.0 - s);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// exact_solution (burgers.py:109-127) -> (u, v)
__device__ inline void exact_uv(double a, double lam, double x, double y, double nu,
                                double& u, double& v) {
  const double ep = exp(lam * (x - 1.0));
  const double em = exp(-lam * (x - 1.0));
  const double cy = cos(lam * y);
  const double sy = sin(lam * y);
  const double psi = a * (1.0 + x) + (ep + em) * cy;
  u = -2.0 * nu * (a + lam * (ep - em) * cy) / psi;
  v = 2.0 * nu * lam * (ep + em) * sy / psi;
}

// boundary values (bx, by, c) of assemble() at every sampled row
// (burgers.py:188-210): ghost points just outside the edges the node touches.
__device__ inline void row_bvals(const Params& P, const StRows& RW, int row, double a, double lm, double* out) {
  const double hx = P.hx, hy = P.hy, nu = P.nu;
  const int bflags = RW.bflags[row];
  const double xc = RW.xc[row], yc = RW.yc[row];
  const bool isv = (bflags >> 4) & 1;
  double exl = 0.0, exr = 0.0, eyb = 0.0, eyt = 0.0, u, v;
  if (bflags & 1) { exact_uv(a, lm, -1.0, yc, nu, u, v); exl = isv ? v : u; }
  if (bflags & 2) { exact_uv(a, lm, 1.0, yc, nu, u, v); exr = isv ? v : u; }
  if (bflags & 4) { exact_uv(a, lm, xc, 0.0, nu, u, v); eyb = isv ? v : u; }
  if (bflags & 8) { exact_uv(a, lm, xc, 0.05, nu, u, v); eyt = isv ? v : u; }
  out[0] = (-1.0 / (2.0 * hx)) * (exl - exr);
  out[1] = (-1.0 / (2.0 * hy)) * (eyb - eyt);
  out[2] = (nu / (hx * hx)) * (exl + exr) + (nu / (hy * hy)) * (eyb + eyt);
}

}  // namespace ddnm
