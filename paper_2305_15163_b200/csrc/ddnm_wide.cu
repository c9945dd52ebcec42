// Batch-wide evaluation kernels (one lane per mu): see ddnm_wide.h.
#include "ddnm_wide.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace ddnm {

// --------------------------------------------------------------------------
// device tables

#ifndef DDNM_WIDE_HU
#define DDNM_WIDE_HU 2             // hidden units computed together (unroll of the activation chain)
#endif
#ifndef DDNM_WIDE_SU
#define DDNM_WIDE_SU 2             // sweep steps unrolled
#endif
constexpr int WIDE_HU = DDNM_WIDE_HU, WIDE_SU = DDNM_WIDE_SU;
constexpr int WRING = 32;          // hidden units a warp keeps in its ring
constexpr int WDEC_WARPS = 12;     // warps per decoder CTA (16 KB ring each)
constexpr int WROW_THREADS = 128;
constexpr int WROW_CHUNK = 32;     // sampled rows per Gram partial
constexpr int WCON_CHUNK = 64;     // interface outputs per constraint partial

// outputs a sweep tile carries at once (register tile of T x (L + 1) sums)
__host__ __device__ constexpr int wide_tile_outputs(int L) { return L <= 8 ? 4 : 2; }

// a tile: up to T consecutive outputs whose hidden windows fit one ring;
// [klo, khi) is the union of their windows, soff the offset of its W2 stream
// ([khi - klo][T] doubles, 0 where an output's window does not hold k)
struct WTile { int o0, cnt, klo, khi, soff; };

struct WDecDev {
  int L, n_out, n_hidden, xoff, act, gj_off;
  const double* W1p;     // [n_hidden][LP], LP = L rounded up to even (uniform row loads)
  const double* b1;
  const double* scale;
  const double* shift;
  const WTile* tiles;
  const double* w2;
};

// one sampled row's tables (RestrictedResidual, partition.py:372-425), 256 bytes:
// source codes of its <= 6 columns (>= 0 interior output, < 0: -1 - interface
// output; padded with the node's own column and zero coefficients), of the
// node's (u, v), its entry count, and the Bx / By / Cdiff coefficients
struct WRowMeta {
  int c[MAXE];
  int cu, cv, ne, pad;
  double bxc[MAXE], byc[MAXE], cdc[MAXE];
  double pad2[9];
};
static_assert(sizeof(WRowMeta) == 256, "one record per 32 lanes x 8 bytes");

// Decoder work comes in two granularities: coarse parts when the running mu
// fill the machine by themselves, fine parts (a couple of tiles each) for the
// rounds where few mu are left and the latency of one item is the round's
// time.  An output is computed by one warp in the same order either way, and
// the row / constraint chunks (whose partial sums fix the rounding) are the
// same in every round: a mu's results do not depend on what else is running.
struct WBlockDev {
  WDecDev dec[2];        // interior subnet, interface decoder
  StRows rows;           // the block's sampled rows (device tables of the context)
  int nrows, row_off, eb_off;
  int rc0, n_rc;         // its row chunks (Gram partial slots rc0 ..)
  int cc0, n_cc;         // its constraint chunks
  const double* CAt;     // [N_Gamma][nCp] C A_i transposed, nCp = n_C rounded up to 8
  const WRowMeta* meta;  // [nrows]
};

struct WPart { int blk, which, t0, t1; };     // a run of tiles of one decoder
struct WRowChunk { int blk, r0, r1, pslot; };
struct WConChunk { int blk, j0, j1, cslot; };

constexpr int WSPEC_MAX = 16;     // most step lengths of one mu evaluated in one round
constexpr int WSPEC_BOOST_LANES = 384;   // boost the candidates while the round stays below this

struct WArgs {
  const WBlockDev* blk;
  const WPart* parts[2];      // coarse, fine
  const WRowChunk* rcs;
  const WConChunk* ccs;
  int nb, nparts[2], nrc, ncc;
  // the blocks this call evaluates ([b_lo, b_hi): a rank of a subdomain-sharded
  // solve) as ranges of the part / chunk tables (sorted by block), and where
  // the packets go: by lane (with speculative candidates) or one row per mu
  int b_lo, b_hi, part_lo[2], part_hi[2], rc_lo, rc_hi, cc_lo, cc_hi, by_mu;
  int S;                 // g/J slots per lane
  int NQ;                // doubles per Gram partial: W (W + 1) / 2 + W + 1
  int nC, nCp, NI, NG;
  int B, vpad;           // batch; lane capacity (a multiple of 32)
  int* act;              // [vpad] lane -> mu | candidate << 24
  int* vbase;            // [B] first lane of each running mu
  int* kof;              // [B] its candidates this round
  int* ctl;              // [0] lanes, [1] decoder items, [2] row / constraint items
  unsigned long long* lanes_total;   // evaluations launched since wide_begin (incl. unused candidates)
  unsigned long long* counters;      // [0] block evaluations consumed (by_mu: counted here)
  const double* trial;
  int rec;
  const SlotState* st;   // [B] SQP state (phase, rejected trials, step length)
  const double* vec;     // [B][8][nK] x, lam, s, slam, ...
  int nK;
  double factor;
  int max_halvings;
  int spec;              // 0: one candidate per mu
  double* gj;
  double* part;
  double* conpart;
  double* bvT;
  int bpad;              // mu stride of bvT
  double* packets;       // [lane][pk_stride]
  int pk_stride, eb_base;
};

// lanes of the round -> decoder part granularity (0 coarse, 1 fine): fine parts
// (more items, hidden units at part boundaries computed twice) only while the
// coarse ones would leave warps of the machine without an item
constexpr int WIDE_FILL_ITEMS = 4096;
__device__ __forceinline__ int wide_mode(const WArgs& A, int nlane) {
  return (long long)(A.part_hi[0] - A.part_lo[0]) * ((nlane + 31) >> 5) < WIDE_FILL_ITEMS ? 1 : 0;
}

// --------------------------------------------------------------------------
// compaction + speculation.  Running mu (trial record flag != 0) in ascending
// order, each with K candidate step lengths alpha, alpha f, alpha f^2, ...:
// after a KKT solve the backtracking line search (sqp.py:262-293) tries
// x + alpha s for a fixed sequence of alpha until Armijo holds, so the
// evaluations of later candidates do not depend on earlier ones and can run in
// the same round; k_dd_step then consumes them in order and stops at the first
// accepted one -- the same iterates, n_evals and histories as one candidate
// per round, in fewer rounds.  K doubles with the rejections already seen
// (1, 2, 4, 4, 8, ...), so at most about as many evaluations are wasted as were
// needed; K = 1 for everybody when the lanes would not fit.

__device__ __forceinline__ int wide_kspec(const WArgs& A, const SlotState& S, bool boost) {
  if (!A.spec || A.by_mu || S.phase != PH_TRIAL || S.n_trials == 0) return 1;
  const int left = A.max_halvings + 1 - S.n_trials;      // trials the reference may still run
  int k = S.n_trials == 1 ? 2 : (S.n_trials < 4 ? 4 : 8);
  // few lanes: a round costs its latency, not its lanes, so candidates are free
  if (boost) k = WSPEC_MAX;
  return max(1, min(k, left));
}

// exclusive prefix of one count per thread over the CTA (1024 threads): warp
// shuffles, the 32 warp totals scanned by warp 0; returns the CTA total too
__device__ __forceinline__ int wide_block_scan(int n, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  __syncthreads();                      // s_warp of an earlier scan has been read
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    s_warp[32 + lane] = w;              // inclusive warp totals
  }
  __syncthreads();
  total = s_warp[32 + 31];
  return incl - n + (warp > 0 ? s_warp[32 + warp - 1] : 0);
}

__global__ void __launch_bounds__(1024) k_wide_compact(const WArgs A) {
  __shared__ int s_warp[64];
  const int tid = threadIdx.x, T = blockDim.x;
  const int per = (A.B + T - 1) / T;
  const int lo = min(A.B, tid * per), hi = min(A.B, lo + per);
  // candidates of this thread's mu under each policy: 2 boosted (few lanes),
  // 1 by the rejections seen, 0 one each
  int n[3] = {0, 0, 0};
  for (int mu = lo; mu < hi; ++mu)
    if (A.trial[(size_t)mu * A.rec] != 0.0) {
      const SlotState S = A.st[mu];
      n[0] += 1;
      n[1] += wide_kspec(A, S, false);
      n[2] += wide_kspec(A, S, true);
    }
  int policy = 2, at = 0, total = 0;
  for (; policy >= 0; --policy) {
    at = wide_block_scan(n[policy], s_warp, total);
    if (policy == 0 || total <= (policy == 2 ? min(WSPEC_BOOST_LANES, A.vpad) : A.vpad)) break;
  }
  for (int mu = lo; mu < hi; ++mu)
    if (A.trial[(size_t)mu * A.rec] != 0.0) {
      const int k = policy ? wide_kspec(A, A.st[mu], policy == 2) : 1;
      A.vbase[mu] = at;
      A.kof[mu] = k;
      for (int j = 0; j < k; ++j) A.act[at++] = mu | (j << 24);
    }
  if (tid == T - 1) {
    A.ctl[0] = total;
    A.ctl[1] = 0; A.ctl[2] = 0; A.ctl[3] = 0;
    *A.lanes_total += (unsigned long long)total;
    if (A.by_mu) atomicAdd(A.counters, (unsigned long long)total * (A.b_hi - A.b_lo));
  }
}

// --------------------------------------------------------------------------
// boundary values by mu: bvT[(row * 3 + c) * bpad + mu]  (burgers.py:188-210)

__global__ void k_wide_bv(const __grid_constant__ Params P, double* bvT, int bpad) {
  const int mu = blockIdx.x * blockDim.x + threadIdx.x;
  const int grow = blockIdx.y;
  if (mu >= P.B) return;
  int b = 0;
  while (b + 1 < P.nb && grow >= P.blk[b + 1].row_off) ++b;
  double out[3];
  row_bvals(P, P.blk[b].rows, grow - P.blk[b].row_off, P.mu[2 * mu], P.mu[2 * mu + 1], out);
#pragma unroll
  for (int c = 0; c < 3; ++c) bvT[((size_t)grow * 3 + c) * bpad + mu] = out[c];
}

// --------------------------------------------------------------------------
// decoder: hidden ring + banded sweep, lane = mu

extern __shared__ __align__(16) double2 wide_ring[];

// next work item of a kernel's queue (one atomic per warp)
__device__ __forceinline__ long long wide_next(int* counter) {
  int v = 0;
  if ((threadIdx.x & 31) == 0) v = atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, v, 0);
}

// --- per-warp weight staging (cp.async, double buffered) ---------------------
// A tile's weights -- its W2 stream, the W1 rows and biases of its hidden
// window, the scale/shift of its outputs: at most one ring of rows -- are
// copied global -> shared asynchronously one tile ahead, so the sweep and the
// hidden layer read them as broadcast shared loads and never wait on L2.
// Layout of one buffer (doubles): W2 [32][4] | W1 [32][LPM] | b1 [32] | scale[4] shift[4]
__host__ __device__ constexpr int wide_lp(int L) { return (L + 1) & ~1; }
__host__ __device__ constexpr int wide_stage_doubles(int lpm) { return 128 + 32 * lpm + 32 + 8; }
// doubles of shared memory per decoder warp: ring (32 x 32 double2) + 2 buffers
__host__ __device__ constexpr int wide_warp_doubles(int lpm) { return 2 * WRING * 32 + 2 * wide_stage_doubles(lpm); }

__device__ __forceinline__ void wide_cp16(double* smem, const double* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void wide_cp8(double* smem, const double* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void wide_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wide_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct WTileR { int o0, cnt, klo, khi, soff; };
__device__ __forceinline__ WTileR wide_tile_load(const WTile* tp) {
  WTileR t;
  t.o0 = __ldg(&tp->o0); t.cnt = __ldg(&tp->cnt); t.klo = __ldg(&tp->klo);
  t.khi = __ldg(&tp->khi); t.soff = __ldg(&tp->soff);
  return t;
}

template <int L, int LPM>
__device__ __forceinline__ void wide_stage(const WDecDev& D, const WTileR& t, double* buf) {
  constexpr int T = wide_tile_outputs(L), LP = wide_lp(L);
  const int lane = threadIdx.x & 31;
  const int nk = t.khi - t.klo;
  const double* g2 = D.w2 + (size_t)t.soff;
  for (int i = lane; i < nk * (T / 2); i += 32) wide_cp16(buf + 2 * i, g2 + 2 * i);
  const double* g1 = D.W1p + (size_t)t.klo * LP;
  for (int i = lane; i < nk * (LP / 2); i += 32) wide_cp16(buf + 128 + 2 * i, g1 + 2 * i);
  if (lane < nk) wide_cp8(buf + 128 + 32 * LPM + lane, D.b1 + t.klo + lane);
  if (lane < t.cnt) wide_cp8(buf + 128 + 32 * LPM + 32 + lane, D.scale + t.o0 + lane);
  else if (lane >= 4 && lane - 4 < t.cnt) wide_cp8(buf + 128 + 32 * LPM + 32 + lane, D.shift + t.o0 + lane - 4);
  // (scale at [0, 4), shift at [4, 8) of the last 8 doubles)
}

template <int L, int CNT>
__device__ __forceinline__ void wide_sweep(const double2* ring, const double* stg, int klo, int khi,
                                           double (&acc)[wide_tile_outputs(L)][L + 1]) {
  constexpr int T = wide_tile_outputs(L), LP = wide_lp(L);
  const double2* wv = reinterpret_cast<const double2*>(stg);
  const double2* w1 = reinterpret_cast<const double2*>(stg + 128);
#pragma unroll WIDE_SU
  for (int k = klo; k < khi; ++k) {
    const double2 sd = ring[(k & (WRING - 1)) * 32];
    double w[LP], v[T];
#pragma unroll
    for (int i = 0; i < LP / 2; ++i) {
      const double2 t = w1[i];
      w[2 * i] = t.x; w[2 * i + 1] = t.y;
    }
#pragma unroll
    for (int i = 0; i < T / 2; ++i) {
      const double2 t = wv[i];
      v[2 * i] = t.x; v[2 * i + 1] = t.y;
    }
    w1 += LP / 2;
    wv += T / 2;
#pragma unroll
    for (int j = 0; j < CNT; ++j) {
      // g += W2 act, J_d += (W2 act') W1[k, d]   (hyper.py:190-197)
      const double t = v[j] * sd.y;
      acc[j][0] = fma(v[j], sd.x, acc[j][0]);
#pragma unroll
      for (int d = 0; d < L; ++d) acc[j][1 + d] = fma(t, w[d], acc[j][1 + d]);
    }
  }
}

// the point lane (mu, j) evaluates: candidate 0 is the trial record's point
// (x0, x + s or x + alpha s as k_dd_step left it), candidate j > 0 the j-th
// further halving, alpha_j = alpha_{j-1} f and x + alpha_j s rounded exactly as
// slot_decide does when it rejects a trial (sqp.py:283-287)
template <int L>
__device__ __forceinline__ void wide_trial_point(const WArgs& A, int e, int xoff, double (&x)[L]) {
  const int mu = e & 0xffffff, j = e >> 24;
  if (j == 0) {
    const double* xr = A.trial + (size_t)mu * A.rec + 1 + xoff;
#pragma unroll
    for (int d = 0; d < L; ++d) x[d] = xr[d];
  } else {
    double al = A.st[mu].alpha;
    for (int i = 0; i < j; ++i) al = al * A.factor;
    const double* xc = A.vec + (size_t)mu * 8 * A.nK + xoff;
    const double* sv = xc + 2 * A.nK;
#pragma unroll
    for (int d = 0; d < L; ++d) x[d] = __dadd_rn(xc[d], __dmul_rn(al, sv[d]));
  }
}

template <int L, int LPM>
__device__ __forceinline__ void wide_dec_part(const WArgs& A, const WDecDev& D, int t0, int t1,
                                              int tile, int nact, double* wsm) {
  constexpr int T = wide_tile_outputs(L), LP = wide_lp(L), STG = wide_stage_doubles(LPM);
  const int lane = threadIdx.x & 31;
  double2* ring = reinterpret_cast<double2*>(wsm) + lane;
  double* stg0 = wsm + 2 * WRING * 32;
  double x[L];
  wide_trial_point<L>(A, A.act[min(tile * 32 + lane, nact - 1)], D.xoff, x);
  double* out = A.gj + ((size_t)tile * A.S + D.gj_off) * 32 + lane;
  const int act = D.act;
  // tile ti staged in buffer cur, tile ti + 1's record loaded (staged below)
  WTileR m0 = wide_tile_load(D.tiles + t0);
  WTileR m1 = t0 + 1 < t1 ? wide_tile_load(D.tiles + t0 + 1) : m0;
  int next_k = m0.klo, cur = 0;
  __syncwarp();                      // the previous item's reads of the buffers are done
  wide_stage<L, LPM>(D, m0, stg0);
  wide_cp_commit();
  for (int ti = t0; ti < t1; ++ti) {
    const WTileR m2 = ti + 2 < t1 ? wide_tile_load(D.tiles + ti + 2) : m1;
    if (ti + 1 < t1) wide_stage<L, LPM>(D, m1, stg0 + (cur ^ 1) * STG);
    wide_cp_commit();
    wide_cp_wait<1>();
    __syncwarp();
    const double* stg = stg0 + cur * STG;
    const int klo = m0.klo, khi = m0.khi, cnt = m0.cnt;
    // hidden units of the window not in the ring yet: z = b1 + W1 x in latent
    // order (hyper.py:184-188), activation and derivative (autoencoder.py:31-45)
#pragma unroll WIDE_HU
    for (int k = max(next_k, klo); k < khi; ++k) {
      const double2* wr = reinterpret_cast<const double2*>(stg + 128) + (k - klo) * (LP / 2);
      double w[LP];
#pragma unroll
      for (int i = 0; i < LP / 2; ++i) {
        const double2 t = wr[i];
        w[2 * i] = t.x; w[2 * i + 1] = t.y;
      }
      double z = stg[128 + 32 * LPM + (k - klo)];
#pragma unroll
      for (int d = 0; d < L; ++d) z = fma(w[d], x[d], z);
      double a, da;
      act_pair(act, z, a, da, k_exp2_32);
      ring[(k & (WRING - 1)) * 32] = make_double2(a, da);
    }
    next_k = max(next_k, khi);
    double acc[T][L + 1];
#pragma unroll
    for (int j = 0; j < T; ++j)
#pragma unroll
      for (int d = 0; d <= L; ++d) acc[j][d] = 0.0;
    if constexpr (T == 4) {
      if (cnt == 4) wide_sweep<L, 4>(ring, stg, klo, khi, acc);
      else if (cnt == 3) wide_sweep<L, 3>(ring, stg, klo, khi, acc);
      else if (cnt == 2) wide_sweep<L, 2>(ring, stg, klo, khi, acc);
      else wide_sweep<L, 1>(ring, stg, klo, khi, acc);
    } else {
      if (cnt == 2) wide_sweep<L, 2>(ring, stg, klo, khi, acc);
      else wide_sweep<L, 1>(ring, stg, klo, khi, acc);
    }
#pragma unroll
    for (int j = 0; j < T; ++j) {
      if (j >= cnt) break;
      const int o = m0.o0 + j;
      const double scl = stg[128 + 32 * LPM + 32 + j], sh = stg[128 + 32 * LPM + 36 + j];
      double* p = out + (size_t)o * (L + 1) * 32;
      p[0] = __dadd_rn(__dmul_rn(acc[j][0], scl), sh);
#pragma unroll
      for (int d = 0; d < L; ++d) p[(1 + d) * 32] = acc[j][1 + d] * scl;
    }
    __syncwarp();                    // buffer cur is free for the tile after next
    m0 = m1; m1 = m2; cur ^= 1;
  }
  wide_cp_wait<0>();
}

template <int NI, int NG>
__global__ void __launch_bounds__(WDEC_WARPS * 32, 1) k_wide_dec(const __grid_constant__ WArgs A) {
  constexpr int LPM = wide_lp(NI) > wide_lp(NG) ? wide_lp(NI) : wide_lp(NG);
  const int nact = A.ctl[0];
  if (nact <= 0) return;
  const int ntile = (nact + 31) >> 5, mode = wide_mode(A, nact);
  const WPart* parts = A.parts[mode] + A.part_lo[mode];
  const long long total = (long long)(A.part_hi[mode] - A.part_lo[mode]) * ntile;
  double* wsm = reinterpret_cast<double*>(wide_ring) + (size_t)(threadIdx.x >> 5) * wide_warp_doubles(LPM);
  for (long long item = wide_next(A.ctl + 1); item < total; item = wide_next(A.ctl + 1)) {
    const int pi = (int)(item / ntile), tile = (int)(item - (long long)pi * ntile);
    const WPart* pp = parts + pi;
    const int b = __ldg(&pp->blk), which = __ldg(&pp->which), t0 = __ldg(&pp->t0), t1 = __ldg(&pp->t1);
    const WBlockDev& B = A.blk[b];
    if (which == 0) wide_dec_part<NI, LPM>(A, B.dec[0], t0, t1, tile, nact, wsm);
    else wide_dec_part<NG, LPM>(A, B.dec[1], t0, t1, tile, nact, wsm);
  }
}

// --------------------------------------------------------------------------
// sampled rows: residual, stencil Jacobian row, chain rule, Gram partial

// first triangle row of part H of NH (rows split so the parts hold about the
// same number of entries)
__host__ __device__ constexpr int wide_tri_row(int W, int NH, int H) {
  if (H <= 0) return 0;
  if (H >= NH) return W;
  const int total = W * (W + 1) / 2;
  int acc = 0, i = 0;
  while (i < W && acc * NH < total * H) { acc += W - i; ++i; }
  return i;
}
__host__ __device__ constexpr int wide_tri_count(int W, int i0, int i1) {
  int n = 0;
  for (int i = i0; i < i1; ++i) n += W - i;
  return n;
}

// A CTA (4 warps) takes one chunk of rows for one lane tile: warp w sums its
// quarter of the rows in row order, then warp 0 adds the quarters in order, so
// a chunk's partial is ((q0 + q1) + q2) + q3 whatever else the round runs.
template <int NI, int NG, int NH, int H>
__device__ __forceinline__ void wide_rows_body(const WArgs& A, const WBlockDev& B, int c0, int c1,
                                               int pslot, int tile, int nact, double* red) {
  constexpr int W = NI + NG;
  constexpr int I0 = wide_tri_row(W, NH, H), I1 = wide_tri_row(W, NH, H + 1);
  constexpr int NA = wide_tri_count(W, I0, I1);
  constexpr int TRI = W * (W + 1) / 2;
  // the CTA's 4 warps: NSPLIT row splits x NH triangle parts.  With NH = 2
  // the two warps of a split walk the same rows: they share the fetched row
  // (each copies every other line) and synchronise on a named barrier.
  constexpr int NSPLIT = 4 / NH;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sp = NH == 2 ? warp >> 1 : warp;
  const int r0 = c0 + (c1 - c0) * sp / NSPLIT, r1 = c0 + (c1 - c0) * (sp + 1) / NSPLIT;
  const int pstride = A.vpad;
  const int pos = tile * 32 + lane;
  const int mu = A.act[min(pos, nact - 1)] & 0xffffff;
  const double* gI = A.gj + ((size_t)tile * A.S + B.dec[0].gj_off) * 32 + lane;
  auto pair_sync = [&]() {
    if constexpr (NH == 2) asm volatile("bar.sync %0, 64;" ::"r"(1 + sp) : "memory");
  };
  // offset of an entry's g value from gI (its Jacobian row follows it):
  // interior output c, or interface output -1 - c of the block's second decoder
  const long long goff = (long long)(B.dec[1].gj_off - B.dec[0].gj_off) * 32;
  auto slot = [&](int c) -> long long {
    return c >= 0 ? (long long)c * (NI + 1) * 32 : goff + (long long)(-1 - c) * (NG + 1) * 32;
  };
  constexpr int LM = NI > NG ? NI : NG;
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = 0.0;
  double proj[W];
#pragma unroll
  for (int i = 0; i < W; ++i) proj[i] = 0.0;
  double rr = 0.0;
  // Every value a row needs from memory -- the g of its <= 6 columns and of
  // the node's (u, v), its boundary values, the Jacobian rows of its columns:
  // NSL (= 11 + 6 LM) coalesced 256-byte lines per warp -- has an address that
  // depends on the row only, so row r + 1 is fetched into shared memory with
  // cp.async (each lane its own 8 bytes of every line) while row r is computed:
  // ~90 lines in flight per warp instead of what fits in registers.  A lane
  // reads back only what it copied itself (no warp synchronisation).  Rows
  // are padded to MAXE entries with zero coefficients on a valid column;
  // adding their exact zeros changes no sum.
  constexpr int NSL = 11 + MAXE * LM;
  double* pbuf = red + (size_t)sp * 2 * NSL * 32 + lane;
  // The rows' own tables (columns, coefficients: one 256-byte WRowMeta per row)
  // run two rows further ahead through a 4-deep ring per warp, lane l copying
  // word l: the record of row r + 1 is in shared memory when its lines are
  // requested, and nothing in the loop waits on a global load.
  double* mring = red + (size_t)NSPLIT * 2 * NSL * 32 + (size_t)warp * 4 * 32;
  const double* mglob = reinterpret_cast<const double*>(B.meta);
  auto fetch_meta = [&](int it) {
    if (it < r1) wide_cp8(mring + ((it - r0) & 3) * 32 + lane, mglob + (size_t)it * 32 + lane);
  };
  auto meta_of = [&](int it) { return reinterpret_cast<const WRowMeta*>(mring + ((it - r0) & 3) * 32); };
  // this warp's share of a row's lines: all of them, or every other one
  auto mine = [&](int line) { return NH == 1 || (line & 1) == H; };
  auto fetch = [&](int it, double* buf) {
    const WRowMeta* m = meta_of(it);
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int ce = m->c[e];
      const double* src = gI + slot(ce);
      if (mine(e)) wide_cp8(buf + e * 32, src);
      const int le = ce >= 0 ? NI : NG;
#pragma unroll
      for (int d = 0; d < LM; ++d)
        if (d < le && mine(11 + e * LM + d)) wide_cp8(buf + (11 + e * LM + d) * 32, src + (1 + d) * 32);
    }
    if (mine(6)) wide_cp8(buf + 6 * 32, gI + slot(m->cu));
    if (mine(7)) wide_cp8(buf + 7 * 32, gI + slot(m->cv));
    const double* bvp = A.bvT + (size_t)(B.row_off + it) * 3 * A.bpad + mu;
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (mine(8 + i)) wide_cp8(buf + (8 + i) * 32, bvp + (size_t)i * A.bpad);
  };
  fetch_meta(r0); fetch_meta(r0 + 1); fetch_meta(r0 + 2);
  wide_cp_commit();
  wide_cp_wait<0>();
  __syncwarp();
  if (r0 < r1) fetch(r0, pbuf);
  wide_cp_commit();
  for (int row = r0; row < r1; ++row) {
    const int par = (row - r0) & 1;
    pair_sync();                       // the pair is done with the row before (its buffer is refilled now)
    if (row + 1 < r1) fetch(row + 1, pbuf + (par ^ 1) * NSL * 32);
    fetch_meta(row + 3);
    wide_cp_commit();
    wide_cp_wait<1>();                 // row's lines and the record of row + 2 have landed
    __syncwarp();
    pair_sync();                       // both halves of this row have landed
    const double* buf = pbuf + par * NSL * 32;
    const WRowMeta* m = meta_of(row);
    const int ne = m->ne, cu = m->cu, cv = m->cv;
    int c[MAXE];
    double bxc[MAXE], byc[MAXE], cdc[MAXE], xe[MAXE];
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      c[e] = m->c[e];
      bxc[e] = m->bxc[e];
      byc[e] = m->byc[e];
      cdc[e] = m->cdc[e];
      xe[e] = buf[e * 32];
    }
    const double xu = buf[6 * 32], xv = buf[7 * 32];
    const double bx = buf[8 * 32], by = buf[9 * 32], bc = buf[10 * 32];
    // xu (Bx x - bx) + xv (By x - by) + Cd x + c   (partition.py:434-441)
    double sx = 0.0, sy = 0.0, scd = 0.0;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      sx = __dadd_rn(sx, __dmul_rn(bxc[e], xe[e]));
      sy = __dadd_rn(sy, __dmul_rn(byc[e], xe[e]));
      scd = __dadd_rn(scd, __dmul_rn(cdc[e], xe[e]));
    }
    const double tx = sx - bx, ty = sy - by;
    const double r = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(xu, tx), __dmul_rn(xv, ty)), scd), bc);
    double R[W];
#pragma unroll
    for (int d = 0; d < W; ++d) R[d] = 0.0;
    // chain rule, the Jacobian row of entry e + 1 read while entry e is used
    double vn[LM];
#pragma unroll
    for (int d = 0; d < LM; ++d) vn[d] = d < (c[0] >= 0 ? NI : NG) ? buf[(11 + d) * 32] : 0.0;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      double v[LM];
#pragma unroll
      for (int d = 0; d < LM; ++d) v[d] = vn[d];
      if (e + 1 < MAXE) {
#pragma unroll
        for (int d = 0; d < LM; ++d)
          vn[d] = d < (c[e + 1] >= 0 ? NI : NG) ? buf[(11 + (e + 1) * LM + d) * 32] : 0.0;
      }
      // diag(Bx x - b) E_u + diag(x_u) Bx + diag(x_v) By + diag(By x - b) E_v + Cd
      double j = 0.0;
      if (c[e] == cu) j = tx;
      if (c[e] == cv) j = __dadd_rn(j, ty);
      j = __dadd_rn(j, __dmul_rn(xu, bxc[e]));
      j = __dadd_rn(j, __dmul_rn(xv, byc[e]));
      j = __dadd_rn(j, cdc[e]);
      if (e >= ne) j = 0.0;
      if (c[e] >= 0) {
#pragma unroll
        for (int d = 0; d < NI; ++d) R[d] = fma(j, v[d], R[d]);
      } else {
#pragma unroll
        for (int d = 0; d < NG; ++d) R[NI + d] = fma(j, v[d], R[NI + d]);
      }
    }
    // H += R^T R (rows I0 .. I1 of the upper triangle), R^T r, r^T r
    {
      int q = 0;
#pragma unroll
      for (int i = I0; i < I1; ++i)
#pragma unroll
        for (int jj = i; jj < W; ++jj) { acc[q] = fma(R[i], R[jj], acc[q]); ++q; }
    }
    if (H == 0) {
#pragma unroll
      for (int i = 0; i < W; ++i) proj[i] = fma(R[i], r, proj[i]);
      rr = fma(r, r, rr);
    }
  }
  constexpr int NRM = TRI + W + 1;                   // room of one (split, part) region
  wide_cp_wait<0>();
  __syncthreads();                                   // the reduction scratch aliases the row buffers
  if (sp > 0) {
    double* mine = red + (size_t)((sp - 1) * NH + H) * NRM * 32 + lane;
#pragma unroll
    for (int q = 0; q < NA; ++q) mine[q * 32] = acc[q];
    if (H == 0) {
#pragma unroll
      for (int i = 0; i < W; ++i) mine[(NA + i) * 32] = proj[i];
      mine[(NA + W) * 32] = rr;
    }
  }
  __syncthreads();
  if (sp == 0) {
    for (int w = 0; w < NSPLIT - 1; ++w) {
      const double* o = red + (size_t)(w * NH + H) * NRM * 32 + lane;
#pragma unroll
      for (int q = 0; q < NA; ++q) acc[q] = acc[q] + o[q * 32];
      if (H == 0) {
#pragma unroll
        for (int i = 0; i < W; ++i) proj[i] = proj[i] + o[(NA + i) * 32];
        rr = rr + o[(NA + W) * 32];
      }
    }
    double* dst = A.part + (size_t)pslot * A.NQ * pstride + pos;
    constexpr int Q0 = wide_tri_count(W, 0, I0);
#pragma unroll
    for (int q = 0; q < NA; ++q) dst[(size_t)(Q0 + q) * pstride] = acc[q];
    if (H == 0) {
#pragma unroll
      for (int i = 0; i < W; ++i) dst[(size_t)(TRI + i) * pstride] = proj[i];
      dst[(size_t)(TRI + W) * pstride] = rr;
    }
  }
  __syncthreads();
}

// WFPC constraint partials: cval = C A_i g, cjac = C A_i J over a chunk of
// interface outputs (driver.py:371-373), 8 constraint rows at a time; the
// CTA's warps take quarters of the chunk, added in order by warp 0
template <int NG>
__device__ __forceinline__ void wide_con_body(const WArgs& A, const WBlockDev& B, int c0j, int c1j,
                                              int cslot, int tile, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = c0j + (c1j - c0j) * warp / 4, j1 = c0j + (c1j - c0j) * (warp + 1) / 4;
  const int pstride = A.vpad;
  constexpr int NR = 8 * (NG + 1);
  const double* gG = A.gj + ((size_t)tile * A.S + B.dec[1].gj_off) * 32 + lane;
  double* dst = A.conpart + (size_t)cslot * A.nCp * (NG + 1) * pstride + tile * 32 + lane;
  for (int c0 = 0; c0 < A.nCp; c0 += 8) {
    double acc[8][NG + 1];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int d = 0; d <= NG; ++d) acc[i][d] = 0.0;
#pragma unroll 2
    for (int j = j0; j < j1; ++j) {
      double v[NG + 1];
#pragma unroll
      for (int d = 0; d <= NG; ++d) v[d] = gG[((size_t)j * (NG + 1) + d) * 32];
      const double2* ca = reinterpret_cast<const double2*>(B.CAt + (size_t)j * A.nCp + c0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 t = __ldg(ca + i);
#pragma unroll
        for (int d = 0; d <= NG; ++d) {
          acc[2 * i][d] = fma(t.x, v[d], acc[2 * i][d]);
          acc[2 * i + 1][d] = fma(t.y, v[d], acc[2 * i + 1][d]);
        }
      }
    }
    if (warp > 0) {
      double* mine = red + (size_t)(warp - 1) * NR * 32 + lane;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int d = 0; d <= NG; ++d) mine[(i * (NG + 1) + d) * 32] = acc[i][d];
    }
    __syncthreads();
    if (warp == 0) {
      for (int w = 0; w < 3; ++w) {
        const double* o = red + (size_t)w * NR * 32 + lane;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int d = 0; d <= NG; ++d) acc[i][d] = acc[i][d] + o[(i * (NG + 1) + d) * 32];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int d = 0; d <= NG; ++d)
          dst[(size_t)((c0 + i) * (NG + 1) + d) * pstride] = acc[i][d];
    }
    __syncthreads();
  }
}

extern __shared__ __align__(16) double wide_red[];

// CTA items: row chunks (x NH triangle parts) first, then the constraint chunks
template <int NI, int NG, int NH>
__global__ void __launch_bounds__(WROW_THREADS, 2) k_wide_rows(const __grid_constant__ WArgs A) {
  const int nact = A.ctl[0];
  if (nact <= 0) return;
  __shared__ int s_item;
  const int ntile = (nact + 31) >> 5;
  const int nrow_items = A.rc_hi - A.rc_lo;
  const long long total = (long long)(nrow_items + A.cc_hi - A.cc_lo) * ntile;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(A.ctl + 2, 1);
    __syncthreads();
    const long long item = s_item;
    __syncthreads();
    if (item >= total) break;
    const int ci = (int)(item / ntile), tile = (int)(item - (long long)ci * ntile);
    if (ci < nrow_items) {
      const WRowChunk* rc = A.rcs + A.rc_lo + ci;
      const int b = __ldg(&rc->blk), r0 = __ldg(&rc->r0), r1 = __ldg(&rc->r1), ps = __ldg(&rc->pslot);
      const WBlockDev& B = A.blk[b];
      // (NH = 2: warps 0, 2 take the first triangle part, warps 1, 3 the second)
      if (NH == 1 || ((threadIdx.x >> 5) & 1) == 0) wide_rows_body<NI, NG, NH, 0>(A, B, r0, r1, ps, tile, nact, wide_red);
      else wide_rows_body<NI, NG, NH, NH - 1>(A, B, r0, r1, ps, tile, nact, wide_red);
    } else {
      const WConChunk* cc = A.ccs + A.cc_lo + (ci - nrow_items);
      const int b = __ldg(&cc->blk), j0 = __ldg(&cc->j0), j1 = __ldg(&cc->j1), cs = __ldg(&cc->cslot);
      wide_con_body<NG>(A, A.blk[b], j0, j1, cs, tile, wide_red);
    }
  }
}

// --------------------------------------------------------------------------
// partials -> packets (the block pieces of an evaluation buffer, in the layout
// k_dd_eval writes: H triangle | R^T r | cval | cjac | r^T r), chunk order

__global__ void __launch_bounds__(128) k_wide_pack(const WArgs A) {
  const int nact = A.ctl[0];
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nact) return;
  const int b = A.b_lo + blockIdx.y;
  const WBlockDev& B = A.blk[b];
  const int pstride = A.vpad;
  const int W = A.NI + A.NG, TRI = W * (W + 1) / 2, NG = A.NG, nC = A.nC;
  const int n_rc = B.n_rc, rc0 = B.rc0, n_cc = B.n_cc, cc0 = B.cc0;
  const size_t prow = A.by_mu ? (size_t)(A.act[pos] & 0xffffff) : (size_t)pos;
  double* dst = A.packets + prow * A.pk_stride + (B.eb_off - A.eb_base);
  const int nq = A.NQ + nC * (NG + 1);
  for (int q = blockIdx.z; q < nq; q += gridDim.z) {
    double v = 0.0;
    if (q < A.NQ) {
      for (int k = 0; k < n_rc; ++k) v = v + A.part[((size_t)(rc0 + k) * A.NQ + q) * pstride + pos];
      // q < TRI + W: H then R^T r, contiguous; r^T r goes after cval / cjac
      dst[q < TRI + W ? q : TRI + W + nC + nC * NG] = v;
    } else {
      const int cq = q - A.NQ, c = cq / (NG + 1), d = cq - c * (NG + 1);
      for (int k = 0; k < n_cc; ++k)
        v = v + A.conpart[((size_t)(cc0 + k) * A.nCp * (NG + 1) + cq) * pstride + pos];
      if (d == 0) dst[TRI + W + c] = v;
      else dst[TRI + W + nC + c * NG + (d - 1)] = v;
    }
  }
}

// --------------------------------------------------------------------------
// host side

struct WideKernels {
  int ni, ng;
  const void* dec;
  const void* rows;
  int nh;
};

#define DDNM_WIDE_ENTRY(NI, NG, NH) \
  WideKernels{NI, NG, (const void*)&k_wide_dec<NI, NG>, (const void*)&k_wide_rows<NI, NG, NH>, NH}

static const WideKernels* wide_kernels(int ni, int ng) {
  static const WideKernels table[] = {
      DDNM_WIDE_ENTRY(6, 4, 1), DDNM_WIDE_ENTRY(8, 5, 2), DDNM_WIDE_ENTRY(4, 3, 1),
      DDNM_WIDE_ENTRY(4, 2, 1), DDNM_WIDE_ENTRY(6, 3, 1), DDNM_WIDE_ENTRY(8, 4, 2),
      DDNM_WIDE_ENTRY(10, 5, 2),
  };
  for (const auto& k : table)
    if (k.ni == ni && k.ng == ng) return &k;
  return nullptr;
}

struct Wide {
  std::vector<void*> allocs;
  WArgs A{};
  const WideKernels* K = nullptr;
  int sms = 0;
  int total_rows = 0;
  size_t ring_smem = 0, red_smem = 0;
  int dec_warps = WDEC_WARPS;
  // first part (coarse / fine), row chunk and constraint chunk of every block (+ end)
  std::vector<int> part0[2], rc0, cc0;
  ~Wide() {
    for (void* p : allocs) cudaFree(p);
  }
};

void WideBuffers::release() {
  for (void* p : {(void*)gj, (void*)part, (void*)conpart, (void*)bvT, (void*)act, (void*)ctl,
                  (void*)vbase, (void*)kof, (void*)lanes_total})
    if (p) cudaFree(p);
  *this = WideBuffers{};
}

namespace {
template <typename T>
bool wup(Wide* w, const std::vector<T>& h, const T** d) {
  *d = nullptr;
  if (h.empty()) return true;
  void* p = nullptr;
  if (cudaMalloc(&p, h.size() * sizeof(T)) != cudaSuccess) return false;
  w->allocs.push_back(p);
  if (cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  *d = static_cast<const T*>(p);
  return true;
}
}  // namespace

void wide_free(Wide* w) { delete w; }

// ---- host-only planning (no GPU): tiles, W2 streams, parts, chunks ----------

struct WidePlanDec {
  std::vector<WTile> tiles;
  std::vector<double> w2;       // per tile [khi - klo][T]
  std::vector<int> tile_of;     // tile of every output
  long long steps = 0;          // sum of khi - klo
  long long useful = 0;         // stored W2 entries
};

// why the instance cannot run on the wide engine, or null
static const char* wide_ineligible(const ddnm_artifacts* a) {
  if (getenv("DDNM_NO_WIDE")) return "disabled (DDNM_NO_WIDE)";
  if (a->map_kind != DDNM_MAP_AUTOENCODER) return "linear maps";
  if (a->constraint_mode != DDNM_CON_WFPC) return "SRPC coupling";
  if (!wide_kernels(a->blocks[0].n_int, a->blocks[0].n_gam)) return "latent pair has no wide kernels";
  for (int b = 0; b < a->n_blocks; ++b) {
    if (a->blocks[b].n_basis > 0) return "gappy hyper-reduction";
    if (a->blocks[b].n_int != a->blocks[0].n_int || a->blocks[b].n_gam != a->blocks[0].n_gam)
      return "blocks with different latent dims";
  }
  return nullptr;
}

// sweep tiles of one decoder: up to T consecutive outputs whose windows start
// within 8 hidden units of the first one's and whose union fits the ring
static const char* wide_plan_decoder(const ddnm_decoder& h, int L, WidePlanDec& out) {
  const int T = wide_tile_outputs(L);
  std::vector<int> k0(h.n_out), wd(h.n_out);
  for (int o = 0; o < h.n_out; ++o) {
    wd[o] = (int)(h.indptr[o + 1] - h.indptr[o]);
    k0[o] = wd[o] > 0 ? (int)h.indices[h.indptr[o]] : (o > 0 ? k0[o - 1] : 0);
    for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e)
      if (h.indices[e] != k0[o] + (e - h.indptr[o])) return "decoder rows are not contiguous windows";
    if (wd[o] > WRING) return "decoder row wider than the hidden ring";
    if (o > 0 && k0[o] < k0[o - 1]) return "decoder windows not ascending";
  }
  out.tile_of.assign(h.n_out, -1);
  for (int o = 0; o < h.n_out;) {
    int lo = k0[o], hi = k0[o] + wd[o], cnt = 1;
    while (cnt < T && o + cnt < h.n_out) {
      const int nhi = std::max(hi, k0[o + cnt] + wd[o + cnt]);
      // a joined output must overlap enough to pay for the longer walk
      if (nhi - lo > WRING || k0[o + cnt] - lo > 8) break;
      hi = nhi;
      ++cnt;
    }
    WTile t{o, cnt, lo, hi, (int)out.w2.size()};
    for (int kk = lo; kk < hi; ++kk)
      for (int j = 0; j < T; ++j) {
        double v = 0.0;
        if (j < cnt) {
          const int e = kk - k0[o + j];
          if (e >= 0 && e < wd[o + j]) v = h.data[h.indptr[o + j] + e];
        }
        out.w2.push_back(v);
      }
    for (int j = 0; j < cnt; ++j) {
      out.tile_of[o + j] = (int)out.tiles.size();
      out.useful += wd[o + j];
    }
    out.steps += hi - lo;
    out.tiles.push_back(t);
    o += cnt;
  }
  return nullptr;
}

// parts: runs of ~pt tiles, cut where the windows do not overlap when such a
// cut is near (no hidden unit computed twice)
static void wide_plan_parts(const std::vector<WTile>& tiles, int pt, int b, int which,
                            std::vector<WPart>& parts) {
  const int nt = (int)tiles.size();
  for (int t0 = 0; t0 < nt;) {
    int t1 = std::min(nt, t0 + pt);
    if (t1 < nt && pt >= 4) {
      int best = -1;
      for (int c = std::max(t0 + pt / 2, t0 + 1); c <= std::min(nt - 1, t0 + pt + pt / 2); ++c) {
        int hi_prev = 0;
        for (int q = std::max(t0, c - 4); q < c; ++q) hi_prev = std::max(hi_prev, tiles[q].khi);
        if (tiles[c].klo >= hi_prev && (best < 0 || std::abs(c - (t0 + pt)) < std::abs(best - (t0 + pt))))
          best = c;
      }
      if (best > 0) t1 = best;
    }
    parts.push_back(WPart{b, which, t0, t1});
    t0 = t1;
  }
}

static void wide_part_sizes(int (&part_tiles)[2], int& row_chunk, int& con_chunk) {
  part_tiles[0] = 16; part_tiles[1] = 2;
  row_chunk = WROW_CHUNK;
  con_chunk = WCON_CHUNK;
  if (const char* e = getenv("DDNM_WIDE_PART")) part_tiles[0] = std::max(1, atoi(e));
  if (const char* e = getenv("DDNM_WIDE_ROWS")) row_chunk = std::max(4, atoi(e));
}

int wide_build(const ddnm_artifacts* a, const Params& P, const WideHostRows* rows, int sms, Wide** out,
               std::string& why) {
  *out = nullptr;
  if (const char* r = wide_ineligible(a)) { why = r; return 0; }
  const int ni = a->blocks[0].n_int, ng = a->blocks[0].n_gam;
  const WideKernels* K = wide_kernels(ni, ng);
  auto* w = new Wide();
  w->K = K;
  w->sms = sms;
  std::vector<WBlockDev> blocks(a->n_blocks);
  std::vector<WPart> parts[2];
  std::vector<WRowChunk> rcs;
  std::vector<WConChunk> ccs;
  const int nC = a->n_c, nCp = (nC + 7) & ~7;
  int S = 0;
  // tiles per decoder part (coarse / fine), sampled rows per Gram partial,
  // interface outputs per constraint partial
  int part_tiles[2], row_chunk, con_chunk;
  wide_part_sizes(part_tiles, row_chunk, con_chunk);
  auto fail_build = [&](const char* msg) { why = msg; delete w; return 0; };
  for (int b = 0; b < a->n_blocks; ++b) {
    const ddnm_block& k = a->blocks[b];
    WBlockDev& WB = blocks[b];
    std::memset(&WB, 0, sizeof WB);
    for (int m = 0; m < 2; ++m) w->part0[m].push_back((int)parts[m].size());
    w->rc0.push_back((int)rcs.size());
    w->cc0.push_back((int)ccs.size());
    for (int which = 0; which < 2; ++which) {
      const ddnm_decoder& h = which == 0 ? k.interior : k.interface;
      const int L = which == 0 ? ni : ng, LP = (L + 1) & ~1;
      WDecDev& D = WB.dec[which];
      D.L = L; D.n_out = h.n_out; D.n_hidden = h.n_hidden;
      D.xoff = P.blk[b].xoff + (which == 0 ? 0 : ni);
      D.act = which == 0 ? a->activation : a->gam_activation;
      D.gj_off = S;
      S += h.n_out * (L + 1);
      D.b1 = which == 0 ? P.blk[b].in.b1 : P.blk[b].ga.b1;
      D.scale = which == 0 ? P.blk[b].in.scale : P.blk[b].ga.scale;
      D.shift = which == 0 ? P.blk[b].in.shift : P.blk[b].ga.shift;
      WidePlanDec pd;
      if (const char* r = wide_plan_decoder(h, L, pd)) return fail_build(r);
      std::vector<double> w1p((size_t)h.n_hidden * LP, 0.0);
      for (int kk = 0; kk < h.n_hidden; ++kk)
        for (int d = 0; d < L; ++d) w1p[(size_t)kk * LP + d] = h.W1[(size_t)kk * L + d];
      if (!wup(w, w1p, &D.W1p) || !wup(w, pd.tiles, &D.tiles) || !wup(w, pd.w2, &D.w2))
        return delete w, -1;
      for (int m = 0; m < 2; ++m) wide_plan_parts(pd.tiles, part_tiles[m], b, which, parts[m]);
    }
    WB.rows = P.blk[b].rows;
    {
      const WideHostRows& hr = rows[b];
      std::vector<WRowMeta> meta(k.n_rows);
      for (int r = 0; r < k.n_rows; ++r) {
        WRowMeta& m = meta[r];
        std::memset(&m, 0, sizeof m);
        for (int e = 0; e < MAXE; ++e) {
          m.c[e] = hr.src[(size_t)e * k.n_rows + r];
          m.bxc[e] = hr.bxc[(size_t)e * k.n_rows + r];
          m.byc[e] = hr.byc[(size_t)e * k.n_rows + r];
          m.cdc[e] = hr.cdc[(size_t)e * k.n_rows + r];
        }
        m.cu = hr.sgu[r]; m.cv = hr.sgv[r]; m.ne = hr.nent[r];
      }
      if (!wup(w, meta, &WB.meta)) return delete w, -1;
    }
    WB.nrows = k.n_rows;
    WB.row_off = P.blk[b].row_off;
    WB.eb_off = P.blk[b].eb_off;
    const int ngo = k.interface.n_out;
    {
      WB.rc0 = (int)rcs.size();
      const int nrc = (k.n_rows + row_chunk - 1) / row_chunk;
      for (int c = 0; c < nrc; ++c) {
        // equal chunks (180 rows -> 6 x 30)
        const int r0 = (int)((long long)k.n_rows * c / nrc), r1 = (int)((long long)k.n_rows * (c + 1) / nrc);
        rcs.push_back(WRowChunk{b, r0, r1, (int)rcs.size()});
      }
      WB.n_rc = nrc;
      WB.cc0 = (int)ccs.size();
      const int ncc = std::max(1, (ngo + con_chunk - 1) / con_chunk);
      for (int c = 0; c < ncc; ++c) {
        const int j0 = (int)((long long)ngo * c / ncc), j1 = (int)((long long)ngo * (c + 1) / ncc);
        ccs.push_back(WConChunk{b, j0, j1, (int)ccs.size()});
      }
      WB.n_cc = ncc;
    }
    std::vector<double> cat((size_t)ngo * nCp, 0.0);
    for (int c = 0; c < nC; ++c)
      for (int j = 0; j < ngo; ++j) cat[(size_t)j * nCp + c] = k.CA[(size_t)c * ngo + j];
    if (!wup(w, cat, &WB.CAt)) return delete w, -1;
  }
  for (int m = 0; m < 2; ++m) w->part0[m].push_back((int)parts[m].size());
  w->rc0.push_back((int)rcs.size());
  w->cc0.push_back((int)ccs.size());
  WArgs& A = w->A;
  if (!wup(w, blocks, &A.blk) || !wup(w, rcs, &A.rcs) || !wup(w, ccs, &A.ccs)) return delete w, -1;
  for (int m = 0; m < 2; ++m) {
    if (!wup(w, parts[m], &A.parts[m])) return delete w, -1;
    A.nparts[m] = (int)parts[m].size();
  }
  A.nrc = (int)rcs.size();
  A.ncc = (int)ccs.size();
  A.nb = a->n_blocks;
  A.S = S;
  const int W = ni + ng;
  A.NQ = W * (W + 1) / 2 + W + 1;
  A.nC = nC; A.nCp = nCp; A.NI = ni; A.NG = ng;
  A.spec = getenv("DDNM_WIDE_NOSPEC") ? 0 : 1;
  w->total_rows = P.total_rows;
  {
    const int lpm = std::max(wide_lp(ni), wide_lp(ng));
    const size_t per_warp = (size_t)wide_warp_doubles(lpm) * sizeof(double);
    w->dec_warps = (int)std::min<size_t>(WDEC_WARPS, (size_t)(227 * 1024 - 1024) / per_warp);
    if (const char* e = getenv("DDNM_WIDE_DEC_WARPS")) w->dec_warps = std::max(1, std::min(w->dec_warps, atoi(e)));
    w->ring_smem = per_warp * w->dec_warps;
  }
  // reduction scratch of a row / constraint CTA, aliased with its row buffers
  {
    const int nh = K->nh, nsplit = 4 / nh;
    const size_t rowbuf = (size_t)nsplit * 2 * (11 + MAXE * std::max(ni, ng)) * 32;
    const size_t meta = (size_t)4 * 4 * 32;               // 4 warps x 4 records
    const size_t reduce = std::max((size_t)(nsplit - 1) * nh * A.NQ, (size_t)3 * 8 * (ng + 1)) * 32;
    w->red_smem = (std::max(rowbuf, reduce) + meta) * sizeof(double);
  }
  if (cudaFuncSetAttribute(K->dec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w->ring_smem) != cudaSuccess ||
      cudaFuncSetAttribute(K->rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w->red_smem) != cudaSuccess)
    return delete w, -1;
  *out = w;
  return 0;
}

// host-only plan summary and the tile of every output (ddnm_wide_plan)
int wide_plan(const ddnm_artifacts* a, int32_t* info, int32_t* tile_of, std::string& why) {
  for (int i = 0; i < 10; ++i) info[i] = 0;
  if (const char* r = wide_ineligible(a)) { why = r; return 0; }
  const int ni = a->blocks[0].n_int, ng = a->blocks[0].n_gam;
  int part_tiles[2], row_chunk, con_chunk;
  wide_part_sizes(part_tiles, row_chunk, con_chunk);
  long long tiles = 0, steps = 0, useful = 0, S = 0, outs = 0;
  int maxu = 0;
  std::vector<WPart> parts[2];
  int nrc = 0, ncc = 0;
  for (int b = 0; b < a->n_blocks; ++b) {
    const ddnm_block& k = a->blocks[b];
    for (int which = 0; which < 2; ++which) {
      const ddnm_decoder& h = which == 0 ? k.interior : k.interface;
      const int L = which == 0 ? ni : ng;
      WidePlanDec pd;
      if (const char* r = wide_plan_decoder(h, L, pd)) { why = r; return 0; }
      for (const WTile& t : pd.tiles) maxu = std::max(maxu, t.khi - t.klo);
      for (int m = 0; m < 2; ++m) wide_plan_parts(pd.tiles, part_tiles[m], b, which, parts[m]);
      if (tile_of)
        for (int o = 0; o < h.n_out; ++o) tile_of[outs + o] = (int32_t)(tiles + pd.tile_of[o]);
      outs += h.n_out;
      tiles += (long long)pd.tiles.size();
      steps += pd.steps * wide_tile_outputs(L);
      useful += pd.useful;
      S += (long long)h.n_out * (L + 1);
    }
    nrc += (k.n_rows + row_chunk - 1) / row_chunk;
    ncc += std::max(1, (k.interface.n_out + con_chunk - 1) / con_chunk);
  }
  info[0] = 1;
  info[1] = (int32_t)tiles;
  info[2] = (int32_t)parts[0].size();
  info[3] = (int32_t)parts[1].size();
  info[4] = nrc;
  info[5] = ncc;
  info[6] = (int32_t)std::min<long long>(steps, INT32_MAX);     // W2 stream slots (tile steps x T)
  info[7] = (int32_t)std::min<long long>(useful, INT32_MAX);    // stored decoder entries
  info[8] = (int32_t)std::min<long long>(S, INT32_MAX);         // g / J doubles per lane
  info[9] = maxu;                                               // longest window union (<= ring)
  return 0;
}

int wide_alloc(const Wide* w, int B, WideBuffers* b, std::string& err) {
  if (b->cap >= B) return 0;
  b->release();
  const int bpad = (B + 31) & ~31;
  // lanes: every mu once plus room for the speculative candidates
  const int vpad = std::max(2 * bpad, 1024);
  const WArgs& A = w->A;
  const size_t tiles = (size_t)vpad / 32;
  const size_t part_n = (size_t)A.nrc * vpad * A.NQ;
  const size_t con_n = (size_t)A.ncc * vpad * A.nCp * (A.NG + 1);
  if (cudaMalloc(&b->gj, tiles * A.S * 32 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&b->part, part_n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&b->conpart, con_n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&b->bvT, (size_t)std::max(w->total_rows, 1) * 3 * bpad * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&b->act, (size_t)vpad * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&b->vbase, (size_t)bpad * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&b->kof, (size_t)bpad * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&b->lanes_total, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&b->ctl, 4 * sizeof(int)) != cudaSuccess) {
    b->release();
    cudaGetLastError();
    err = "cannot allocate the wide evaluation buffers";
    return -1;
  }
  b->cap = B;
  b->bpad = bpad;
  b->vpad = vpad;
  return 0;
}

int wide_begin(const Wide* w, const Params& P, WideBuffers& b, cudaStream_t s) {
  (void)w;
  if (cudaMemsetAsync(b.lanes_total, 0, sizeof(unsigned long long), s) != cudaSuccess) return -1;
  if (P.total_rows == 0) return 0;
  dim3 grid((P.B + 127) / 128, P.total_rows);
  k_wide_bv<<<grid, 128, 0, s>>>(P, b.bvT, b.bpad);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int wide_eval(const Wide* w, const Params& P, WideBuffers& b, double* packets, int pk_stride,
              bool by_mu, cudaStream_t s) {
  WArgs A = w->A;
  A.b_lo = P.b_lo;
  A.b_hi = P.b_hi;
  for (int m = 0; m < 2; ++m) { A.part_lo[m] = w->part0[m][P.b_lo]; A.part_hi[m] = w->part0[m][P.b_hi]; }
  A.rc_lo = w->rc0[P.b_lo]; A.rc_hi = w->rc0[P.b_hi];
  A.cc_lo = w->cc0[P.b_lo]; A.cc_hi = w->cc0[P.b_hi];
  A.by_mu = by_mu ? 1 : 0;
  A.B = P.B;
  A.vpad = b.vpad;
  A.bpad = b.bpad;
  A.act = b.act;
  A.vbase = b.vbase;
  A.kof = b.kof;
  A.ctl = b.ctl;
  A.lanes_total = b.lanes_total;
  A.counters = P.counters;
  A.trial = P.dd_trial;
  A.rec = P.dd_rec;
  A.st = P.dd_st;
  A.vec = P.dd_vec;
  A.nK = P.nK;
  A.factor = P.cfg.factor;
  A.max_halvings = P.cfg.max_halvings;
  A.gj = b.gj;
  A.part = b.part;
  A.conpart = b.conpart;
  A.bvT = b.bvT;
  A.packets = packets;
  A.pk_stride = pk_stride;
  A.eb_base = P.blk[P.b_lo].eb_off;
  // DDNM_WIDE_SYNC=1: synchronise after every kernel and name the one that failed
  static const bool dbg = getenv("DDNM_WIDE_SYNC") != nullptr;
  auto chk = [&](const char* what) {
    if (!dbg) return true;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) fprintf(stderr, "ddnm wide: %s failed: %s\n", what, cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  if (!chk("before compact")) return -1;
  k_wide_compact<<<1, 1024, 0, s>>>(A);
  if (!chk("k_wide_compact")) return -1;
  void* args[] = {&A};
  const int ctas = w->sms;
  if (cudaLaunchKernel(w->K->dec, dim3(ctas), dim3(w->dec_warps * 32), args, w->ring_smem, s) != cudaSuccess)
    return -1;
  if (!chk("k_wide_dec")) return -1;
  if (cudaLaunchKernel(w->K->rows, dim3(ctas * 2), dim3(WROW_THREADS), args, w->red_smem, s) != cudaSuccess)
    return -1;
  if (!chk("k_wide_rows")) return -1;
  // lanes of the round are only known on the device: the grid covers the
  // capacity the host can bound (mu still running x candidates)
  const int lanes = std::min(b.vpad, b.lane_bound > 0 ? b.lane_bound : b.vpad);
  dim3 pg((lanes + 127) / 128, A.b_hi - A.b_lo, 16);
  k_wide_pack<<<pg, 128, 0, s>>>(A);
  if (!chk("k_wide_pack")) return -1;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace ddnm

extern "C" int ddnm_wide_plan(const ddnm_artifacts* a, int32_t* info10, int32_t* tile_of_output) {
  if (!a || !info10) { ddnm::set_error("null argument"); return DDNM_EINVAL; }
  if (a->abi_version != DDNM_ABI_VERSION) { ddnm::set_error("ABI version mismatch"); return DDNM_EINVAL; }
  if (a->n_blocks < 1 || a->n_blocks > ddnm::MAXB) { ddnm::set_error("need 1..16 blocks"); return DDNM_EINVAL; }
  std::string why;
  const int rc = ddnm::wide_plan(a, info10, tile_of_output, why);
  ddnm::set_error(why);
  return rc;
}

