// Batch-wide evaluation of eval_gradients (sqp.py:117-146): one lane per mu.
//
// The persistent kernel (ddnm_solve.cuh) gives every mu a slot of one CTA, so
// a weight is shared by the 4 slots of that CTA.  The wide evaluation turns
// the batch sideways: a warp holds 32 running mu in its lanes and walks a run
// of decoder outputs, so every weight, index and stencil coefficient is a
// warp-uniform load shared by 32 mu and every per-mu value is a coalesced
// 256-byte row.  One SQP round of the batch is then
//   k_wide_compact  running mu -> dense lane list (the trial records' flags),
//                   with the line search's next step lengths as extra lanes
//   k_wide_dec      hidden layer (a 32-unit ring per warp in shared memory,
//                   weights staged by cp.async) + banded output sweep, g and
//                   its latent Jacobian (hyper.py:184-197)
//                   -> g/J lines [tile][slot][32 lanes]
//   k_wide_rows     HR stencil rows (prefetched by cp.async), chain rule, Gram
//                   partials per row chunk (partition.py:427-464,
//                   driver.py:422-429, sqp.py:124-133); WFPC constraint
//                   partials C A_i g, C A_i J (driver.py:371-373)
//   k_wide_pack     partials summed in chunk order -> the packets that
//                   k_dd_step (the SQP decision + KKT of ddnm_solve.cuh) reads
// i.e. it replaces k_dd_eval in the round-synchronous solve.
#pragma once
#include <string>

#include <cuda_runtime.h>

#include "../../include/ddnm.h"
#include "ddnm_device.cuh"

namespace ddnm {

void set_error(const std::string& msg);   // ddnm_abi.cu: the thread's ddnm_last_error

// host copy of one block's sampled rows (build_stencil), entry e of row r at [e * nrows + r]
struct WideHostRows {
  const int *src, *sgu, *sgv, *nent;
  const double *bxc, *byc, *cdc;
};

struct Wide;   // the wide program of one instance (device tables)

// scratch of one solve of up to `cap` mu
struct WideBuffers {
  int cap = 0;
  int bpad = 0;               // mu capacity (multiple of 32)
  int vpad = 0;               // lane capacity: running mu x speculative candidates
  int lane_bound = 0;         // host bound on the lanes of the next round (0: vpad)
  double* gj = nullptr;       // [tiles][S][32] decoder values and Jacobian rows
  double* part = nullptr;     // [row chunks][NQ][lanes] Gram partials
  double* conpart = nullptr;  // [con chunks][nCp * (NG + 1)][lanes]
  double* bvT = nullptr;      // [total_rows][3][bpad] boundary values, by mu
  int* act = nullptr;         // [vpad] lane -> mu | candidate << 24
  int* vbase = nullptr;       // [bpad] first lane of a running mu
  int* kof = nullptr;         // [bpad] its candidates this round
  int* ctl = nullptr;         // [0] lanes, [1..3] work counters
  unsigned long long* lanes_total = nullptr;   // evaluations launched this solve
  void release();
};

// *out stays null (return 0) when the instance is not eligible (why says so)
int wide_build(const ddnm_artifacts* a, const Params& P, const WideHostRows* rows, int sms,
               Wide** out, std::string& why);
void wide_free(Wide* w);
int wide_alloc(const Wide* w, int B, WideBuffers* b, std::string& err);
// boundary values of every mu of the batch (once per solve)
int wide_begin(const Wide* w, const Params& P, WideBuffers& b, cudaStream_t s);
// one evaluation of blocks [P.b_lo, P.b_hi) at every running mu's trial point.
// by_mu = false: packets [lane][pk_stride], a mu's speculative candidates in
// consecutive rows (k_dd_step finds them through dd_vbase / dd_kof); by_mu =
// true: one candidate per mu, packets [mu][pk_stride] as k_dd_eval writes them
// (a rank of a subdomain-sharded solve: the other ranks' state is not here)
int wide_eval(const Wide* w, const Params& P, WideBuffers& b, double* packets, int pk_stride,
              bool by_mu, cudaStream_t s);
// packets the solve must provide: one row per lane
inline size_t wide_packet_rows(const WideBuffers& b) { return (size_t)b.vpad; }

}  // namespace ddnm
