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
  const double* W1;       // AE: [n_hidden][lat]; LINEAR: Phi [n_out][lat]
  const double* b1;       // [n_hidden]
  const int* indptr;      // [n_out+1]
  const int* indices;     // [nnz]
  const double* data;     // [nnz]
  const double* scale;    // [n_out]
  const double* shift;    // [n_out]
  int ell_w;              // ELL width (max nnz per row, padded to 4)
  const double* ell_v;    // [ell_w][n_out] W2 values in storage order, 0-padded
  const int* ell_k;       // [ell_w][n_out] hidden indices, 0-padded
};

// One sampled residual row in local-column form (RestrictedResidual,
// partition.py:372-425).  Entries are sorted by global column, which is the
// storage order of the reference's Bx/By/Cdiff rows, so the per-operator sums
// accumulate in the reference order.
struct StRow {
  int gu, gv;             // local positions of u_p and v_p
  int nent;               // distinct local columns referenced (<= 6)
  int bflags;             // bit0 left, bit1 right, bit2 bottom, bit3 top, bit4 v-row
  int col[MAXE];
  double bxc[MAXE], byc[MAXE], cdc[MAXE];
  double xc, yc;          // node coordinates (ghost points share one of them)
};

struct BlockDev {
  int ni, ng, w;          // latent dims, w = ni + ng
  int nrows, n_io, n_gio;
  int xoff;               // offset of (x_int, x_gam) in the stacked latent
  int row_off;            // offset in concatenated rows (bvals, Br)
  int iout_off, gout_off, R_off, cjac_off, intJ_off, gamJ_off;
  int eb_off;             // offset of this block inside a slot eval buffer
  DecDev in, ga;
  const StRow* rows;
  const int* gio;
  const double* CA;       // [n_c][ga.n_out]
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
  int* work;              // [0]: next mu; [1]: finished CTAs
  unsigned long long* counters;  // [0] block-evals, [1] KKT solves
};

struct SlotState {
  int mu, phase, n_iter, n_trials, n_evals, n_reg, status, need_kkt;
  int lam_given, pad;
  double alpha, merit, obj, best_merit;
};

// ---------------------------------------------------------------------------
// scalar helpers

__device__ __forceinline__ double expit_d(double z) {
  // scipy.special.expit: 1 / (1 + exp(-x))
  return 1.0 / (1.0 + exp(-z));
}

__device__ __forceinline__ void act_pair(int act, double z, double& a, double& da) {
  const double s = expit_d(z);
  if (act == ACT_SWISH) {
    a = z * s;
    da = s * (1.0 + z * (1.0 - s));
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

}  // namespace ddnm
