// C ABI of libddnm.so (include/ddnm.h): context management, host-side setup
// of the device tables (the RestrictedResidual stencil of partition.py:361-425
// in local-column form), kernel planning and launches.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ddnm.h"
#include "ddnm_device.cuh"
#include "ddnm_registry.h"
#include "ddnm_wide.h"

using namespace ddnm;

namespace ddnm {
__global__ void k_fill(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
}  // namespace ddnm

// compiled specialisations live in inst_<ni>_<ng>.cu (built in parallel)
using ddnm::KernelEntry;
#define DDNM_DECL(NI, NG) void register_##NI##_##NG(std::vector<KernelEntry>&);
namespace ddnm {
DDNM_DECL(6, 4)
DDNM_DECL(4, 3)
DDNM_DECL(8, 4)
DDNM_DECL(20, 8)
DDNM_DECL(8, 5)
DDNM_DECL(6, 11)
DDNM_DECL(4, 9)
DDNM_DECL(8, 11)
DDNM_DECL(20, 19)
// the declared extra latent pairs (csrc/latent_dims.txt, generated at build time)
void register_generated(std::vector<KernelEntry>&);
}  // namespace ddnm

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace ddnm {
void set_error(const std::string& msg) { g_err = msg; }

// The dynamic shared-memory limit is an attribute of the kernel function,
// shared by every context of the process that uses the same specialisation:
// only ever raise it, so a context planned with less shared memory cannot
// invalidate the launches of one planned with more.
cudaError_t raise_smem_limit(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& v = cur[{dev, fn}];
  if (bytes <= v) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) v = bytes;
  return e;
}
}  // namespace ddnm

namespace {

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(DDNM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

using Kernels = KernelEntry;

// (n_int, n_gam) pairs with compiled kernels: config 0/2 NM (6,4), config 1
// LS (20,8), configs 3/4 (8,5), the small test instances (4,3), (8,4), and
// the SRPC variants (interface latents = sum of port latents): NM (6,11),
// (4,9), LS (20,19), (8,11).
const std::vector<Kernels>& kernel_table() {
  static const std::vector<Kernels> t = [] {
    std::vector<Kernels> v;
    ddnm::register_6_4(v);
    ddnm::register_4_3(v);
    ddnm::register_8_4(v);
    ddnm::register_20_8(v);
    ddnm::register_8_5(v);
    ddnm::register_6_11(v);
    ddnm::register_4_9(v);
    ddnm::register_8_11(v);
    ddnm::register_20_19(v);
    ddnm::register_generated(v);
    return v;
  }();
  return t;
}

}  // namespace

// device buffers of one subdomain-sharded solve (ddnm_dd_*), sized for up to
// `cap` mu; pooled in the context between solves (allocated once, reused)
struct DdBuffers {
  int cap = 0;
  SlotState* st = nullptr;
  double *vec = nullptr, *ecur = nullptr, *gbv = nullptr, *gJ = nullptr, *gJg = nullptr,
         *kkt_g = nullptr, *eb_g = nullptr, *trials = nullptr;
  int* active = nullptr;
  // batch-wide evaluation (ddnm_wide.h): its scratch and the packets of the
  // in-library round loop
  ddnm::WideBuffers wide;
  double* pk = nullptr;
  size_t pk_len = 0;
  double* kkt_fb = nullptr;         // dense-fallback KKT workspace per mu (wide solve)
  void release() {
    wide.release();
    if (pk) cudaFree(pk);
    if (kkt_fb) cudaFree(kkt_fb);
    for (void* p : {(void*)st, (void*)vec, (void*)ecur, (void*)gbv, (void*)gJ, (void*)gJg,
                    (void*)kkt_g, (void*)eb_g, (void*)trials, (void*)active})
      if (p) cudaFree(p);
    *this = DdBuffers{};
  }
};

struct ddnm_ctx {
  int device = 0;
  int sms = 0;
  Params P{};                 // template params (work fields filled per call)
  Kernels K{};
  int threads = 512;
  int ctas = 0;               // persistent grid
  size_t smem = 0;
  int n_D = 0, n_C = 0, nb = 0;
  int tot_rows = 0, tot_iout = 0, tot_gout = 0, tot_R = 0, tot_cjac = 0, tot_intJ = 0,
      tot_gamJ = 0;
  cudaStream_t stream = nullptr;
  std::vector<void*> allocs;  // weights, tables
  double* gbv = nullptr;      // boundary values per global slot
  double* gJ = nullptr;       // interior Jacobian rows per global slot
  double* gJg = nullptr;      // interface Jacobian rows per global slot
  double* kkt_g = nullptr;    // KKT workspace per global slot (KG kernels)
  size_t kkt_stride = 0;      // doubles per slot, 0: KKT in shared memory
  bool ebg = false;           // evaluation buffers in global memory
  double* eb_g = nullptr;     // [slots][2][eb_size] when ebg
  size_t gbv_slots = 0;
  int* work = nullptr;
  unsigned long long* counters = nullptr;
  unsigned long long last_counters[2] = {0, 0};
  unsigned long long* prof = nullptr;   // device-side phase profiler (env DDNM_PROF=1)
  // host-API staging buffers
  std::map<std::string, std::pair<void*, size_t>> io;
  // full decode (ddnm_ctx_set_full_decoders)
  int map_kind = 0;
  int n_units = 0;            // evaluation units (0: blocks evaluated whole)
  std::vector<DdBuffers> dd_pool;   // buffers of finished sharded solves, for reuse
  ddnm::Wide* wide = nullptr;       // batch-wide evaluation program (null: not eligible)
  // step kernel of the batch-wide solve: shared scratch sized for the
  // block-structured KKT only (the dense fallback gets a global workspace),
  // two CTAs per SM when the specialisation has k_dd_step2
  int engine = 0;                   // DDNM_ENGINE_*: 0 auto, 1 slots (persistent kernel), 2 wide
  long long last_rounds = 0, last_launches = 0;   // of the last batched solve
  long long last_lanes = 0;         // evaluations launched by the wide engine (incl. unused candidates)
  int step_scr = 0;                 // doubles per slot (0: use the planner's plan)
  size_t step_smem = 0;
  size_t kkt_fb_stride = 0;
  std::string wide_why;             // why not
  DecodeJob* d_jobs = nullptr;
  int state_len = 0, dec_max_hidden = 0, dec_mu_tile = 0;
};

namespace ddnm {
size_t decode_smem(int mu, int max_hidden);
int decode_mu_tile(int max_hidden, size_t smem_cap);
cudaError_t launch_decode(const DecodeParams& p, cudaStream_t s);
}  // namespace ddnm

namespace {

template <typename T>
int upload(ddnm_ctx* c, const T* h, size_t n, T** d) {
  *d = nullptr;
  if (n == 0) return 0;
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, n * sizeof(T)));
  c->allocs.push_back(p);
  CUDA_TRY(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  *d = static_cast<T*>(p);
  return 0;
}

int upload_i32(ddnm_ctx* c, const int64_t* h, size_t n, int** d) {
  std::vector<int> v(n);
  for (size_t i = 0; i < n; ++i) {
    if (h[i] < INT32_MIN || h[i] > INT32_MAX) return fail(DDNM_EINVAL, "index out of int32 range");
    v[i] = (int)h[i];
  }
  return upload(c, v.data(), n, d);
}

int io_buf(ddnm_ctx* c, const std::string& name, size_t bytes, void** p) {
  auto it = c->io.find(name);
  if (it != c->io.end() && it->second.second >= bytes) {
    *p = it->second.first;
    return 0;
  }
  if (it != c->io.end()) cudaFree(it->second.first);
  void* q = nullptr;
  CUDA_TRY(cudaMalloc(&q, std::max<size_t>(bytes, 8)));
  c->io[name] = {q, bytes};
  *p = q;
  return 0;
}

// RestrictedResidual rows (partition.py:361-425) in local-column form, SoA.
struct HostRows {
  std::vector<int> gu, gv, nent, bflags, col, src, sgu, sgv;
  std::vector<double> bxc, byc, cdc, xc, yc;
};

int build_stencil(const ddnm_artifacts* a, const ddnm_block& blk, HostRows& out) {
  const int nx = a->nx, ny = a->ny;
  const int n = nx * ny;
  const double hx = 2.0 / (nx + 1), hy = 0.05 / (ny + 1), nu = a->nu;
  const double cx = -1.0 / (2.0 * hx), cyy = -1.0 / (2.0 * hy);
  const double dx = nu / (hx * hx), dy = nu / (hy * hy);
  std::vector<int> lookup(2 * (size_t)n, -1);
  for (int k = 0; k < blk.n_cols; ++k) {
    const int64_t c = blk.cols[k];
    if (c < 0 || c >= 2 * (int64_t)n) return fail(DDNM_EINVAL, "column index out of range");
    lookup[c] = k;
  }
  const int nr = blk.n_rows;
  out.gu.assign(nr, 0); out.gv.assign(nr, 0); out.nent.assign(nr, 0); out.bflags.assign(nr, 0);
  out.col.assign((size_t)MAXE * nr, 0);
  out.bxc.assign((size_t)MAXE * nr, 0.0); out.byc.assign((size_t)MAXE * nr, 0.0);
  out.cdc.assign((size_t)MAXE * nr, 0.0);
  out.xc.assign(nr, 0.0); out.yc.assign(nr, 0.0);
  for (int r = 0; r < nr; ++r) {
    const int64_t gr = blk.res_rows[r];
    if (gr < 0 || gr >= 2 * (int64_t)n) return fail(DDNM_EINVAL, "residual row out of range");
    const bool isv = gr >= n;
    const int p = (int)(isv ? gr - n : gr);
    const int off = isv ? n : 0;
    const int i = p % nx, j = p / nx;
    // global column -> (bx, by, cd) coefficients, columns sorted ascending
    std::map<int, std::array<double, 3>> ent;
    auto add = [&](int gc, int which, double w) { ent[gc][which] = w; };
    if (i > 0) add(off + p - 1, 0, cx * -1.0);
    if (i < nx - 1) add(off + p + 1, 0, cx * 1.0);
    if (j > 0) add(off + p - nx, 1, cyy * -1.0);
    if (j < ny - 1) add(off + p + nx, 1, cyy * 1.0);
    if (j > 0) add(off + p - nx, 2, dy * 1.0);
    if (i > 0) add(off + p - 1, 2, dx * 1.0);
    add(off + p, 2, dx * -2.0 + dy * -2.0);
    if (i < nx - 1) add(off + p + 1, 2, dx * 1.0);
    if (j < ny - 1) add(off + p + nx, 2, dy * 1.0);
    ent[isv ? p : n + p];  // cross-component diagonal (E_u / E_v)
    if ((int)ent.size() > MAXE) return fail(DDNM_EINVAL, "stencil row wider than 6");
    out.gu[r] = lookup[p];
    out.gv[r] = lookup[n + p];
    if (out.gu[r] < 0 || out.gv[r] < 0)
      return fail(DDNM_EINVAL, "diagonal coupling column missing from the provided column set");
    int e = 0;
    for (auto& kv : ent) {
      const int lc = lookup[kv.first];
      if (lc < 0)
        return fail(DDNM_EINVAL, "restricted rows reference columns outside the provided column set");
      out.col[(size_t)e * nr + r] = lc;
      out.bxc[(size_t)e * nr + r] = kv.second[0];
      out.byc[(size_t)e * nr + r] = kv.second[1];
      out.cdc[(size_t)e * nr + r] = kv.second[2];
      ++e;
    }
    for (; e < MAXE; ++e) out.col[(size_t)e * nr + r] = out.gu[r];
    out.nent[r] = (int)ent.size();
    out.bflags[r] = (i == 0 ? 1 : 0) | (i == nx - 1 ? 2 : 0) | (j == 0 ? 4 : 0) |
                    (j == ny - 1 ? 8 : 0) | (isv ? 16 : 0);
    out.xc[r] = -1.0 + hx * (i + 1);
    out.yc[r] = hy * (j + 1);
  }
  // source codes: interior outputs keep their index, interface outputs map
  // through gio to -1 - position
  auto code = [&](int c) { return c < blk.n_io ? c : -1 - (int)blk.gio[c - blk.n_io]; };
  out.src.resize(out.col.size());
  for (size_t q = 0; q < out.col.size(); ++q) out.src[q] = code(out.col[q]);
  out.sgu.resize(nr);
  out.sgv.resize(nr);
  for (int r = 0; r < nr; ++r) { out.sgu[r] = code(out.gu[r]); out.sgv[r] = code(out.gv[r]); }
  return 0;
}

int check_decoder(const ddnm_decoder& d, int lat, int kind, const char* what) {
  char buf[160];
  if (d.n_out < 0 || !d.W1) {
    snprintf(buf, sizeof buf, "%s decoder: missing weights", what);
    return fail(DDNM_EINVAL, buf);
  }
  if (kind == DDNM_MAP_AUTOENCODER && d.n_out == 0) return 0;   // empty restriction (no gio)
  if (kind == DDNM_MAP_AUTOENCODER) {
    if (d.n_hidden <= 0 || !d.b1 || !d.indptr || !d.indices || !d.data || !d.scale || !d.shift) {
      snprintf(buf, sizeof buf, "%s decoder: incomplete autoencoder arrays", what);
      return fail(DDNM_EINVAL, buf);
    }
    if (d.indptr[0] != 0) return fail(DDNM_EINVAL, "CSR indptr must start at 0");
    for (int o = 0; o < d.n_out; ++o)
      if (d.indptr[o + 1] < d.indptr[o]) return fail(DDNM_EINVAL, "CSR indptr not monotone");
    const int64_t nnz = d.indptr[d.n_out];
    for (int64_t e = 0; e < nnz; ++e)
      if (d.indices[e] < 0 || d.indices[e] >= d.n_hidden)
        return fail(DDNM_EINVAL, "CSR hidden index out of range");
  }
  (void)lat;
  return 0;
}

struct HostWindows {        // contiguous-window decoders: per-output k0 and width
  std::vector<int> k0, w;
  int maxw = 0;
};

int upload_decoder(ddnm_ctx* c, const ddnm_decoder& h, int lat, int kind, int act, DecDev& d,
                   HostWindows& hw) {
  std::memset(&d, 0, sizeof d);
  d.n_out = h.n_out;
  d.n_hidden = kind == DDNM_MAP_AUTOENCODER ? h.n_hidden : 0;
  d.act = act;
  int rc;
  if (kind == DDNM_MAP_AUTOENCODER && h.n_out == 0) {
    d.n_hidden = 0;      // empty SRPC interface restriction: nothing to evaluate
    return 0;
  }
  if (kind == DDNM_MAP_AUTOENCODER) {
    const size_t nnz = (size_t)h.indptr[h.n_out];
    d.ldw = h.n_hidden + 32;
    std::vector<double> w1t((size_t)d.ldw * lat, 0.0);
    for (int k = 0; k < h.n_hidden; ++k)
      for (int dd = 0; dd < lat; ++dd) w1t[(size_t)dd * d.ldw + k] = h.W1[(size_t)k * lat + dd];
    if ((rc = upload(c, w1t.data(), w1t.size(), const_cast<double**>(&d.W1t)))) return rc;
    d.W1 = nullptr;
    if ((rc = upload(c, h.b1, (size_t)h.n_hidden, const_cast<double**>(&d.b1)))) return rc;
    {   // A fragments of the tensor-core hidden layer (hidden_group)
      const int nt = (h.n_hidden + 7) / 8, ks = (lat + 3) / 4;
      std::vector<double> wa((size_t)nt * ks * 32, 0.0);
      for (int t = 0; t < nt; ++t)
        for (int k = 0; k < ks; ++k)
          for (int l = 0; l < 32; ++l) {
            const int u = 8 * t + (l >> 2), dd = 4 * k + (l & 3);
            if (u < h.n_hidden && dd < lat) wa[((size_t)t * ks + k) * 32 + l] = h.W1[(size_t)u * lat + dd];
          }
      if ((rc = upload(c, wa.data(), wa.size(), const_cast<double**>(&d.w1a)))) return rc;
    }
    if ((rc = upload_i32(c, h.indptr, (size_t)h.n_out + 1, const_cast<int**>(&d.indptr)))) return rc;
    if ((rc = upload_i32(c, h.indices, nnz, const_cast<int**>(&d.indices)))) return rc;
    if ((rc = upload(c, h.data, nnz, const_cast<double**>(&d.data)))) return rc;
    if ((rc = upload(c, h.scale, (size_t)h.n_out, const_cast<double**>(&d.scale)))) return rc;
    if ((rc = upload(c, h.shift, (size_t)h.n_out, const_cast<double**>(&d.shift)))) return rc;
    // ELL-transposed copy of W2 for the sweep (storage order kept per row)
    int64_t wmax = 0;
    for (int o = 0; o < h.n_out; ++o) wmax = std::max<int64_t>(wmax, h.indptr[o + 1] - h.indptr[o]);
    const int ew = (int)((wmax + 7) / 8 * 8);
    std::vector<double> ev((size_t)ew * h.n_out, 0.0);
    std::vector<int> ek((size_t)ew * h.n_out, 0);
    for (int o = 0; o < h.n_out; ++o)
      for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e) {
        const size_t slot = (size_t)(e - h.indptr[o]) * h.n_out + o;
        ev[slot] = h.data[e];
        ek[slot] = (int)h.indices[e];
      }
    d.ell_w = ew;
    // contiguous windows (banded masks, autoencoder.py:76-96): index = k0 + e
    bool contig = true;
    std::vector<int> k0(h.n_out, 0);
    for (int o = 0; o < h.n_out && contig; ++o) {
      if (h.indptr[o + 1] > h.indptr[o]) k0[o] = (int)h.indices[h.indptr[o]];
      for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e)
        if (h.indices[e] != k0[o] + (e - h.indptr[o])) { contig = false; break; }
    }
    d.ell_k = nullptr;
    d.ell_k0 = nullptr;
    d.w1frag = nullptr;
    d.v_row = nullptr;
    d.row_w = nullptr;
    hw.k0.clear();
    hw.w.clear();
    if (ew > 0) {
      ev.push_back(0.0);   // spare zero for masked-out lanes
    if ((rc = upload(c, ev.data(), ev.size(), const_cast<double**>(&d.ell_v)))) return rc;
    d.ell_zero = d.ell_v + ev.size() - 1;
      if (contig) {
        if ((rc = upload(c, k0.data(), k0.size(), const_cast<int**>(&d.ell_k0)))) return rc;
        // tensor-core sweep tables: W1 in A-fragment order, rows contiguous
        const int nkb = (h.n_hidden + 3) / 4;
        std::vector<double> fr((size_t)nkb * 32, 0.0);
        for (int kb = 0; kb < nkb; ++kb)
          for (int l = 0; l < 32; ++l) {
            const int k = 4 * kb + (l & 3), dd = l >> 2;
            if (k < h.n_hidden && dd < lat) fr[(size_t)kb * 32 + l] = h.W1[(size_t)k * lat + dd];
          }
        std::vector<double> vr((size_t)h.n_out * ew, 0.0);
        std::vector<int> rw(h.n_out);
        for (int o = 0; o < h.n_out; ++o) {
          rw[o] = (int)(h.indptr[o + 1] - h.indptr[o]);
          for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e)
            vr[(size_t)o * ew + (e - h.indptr[o])] = h.data[e];
        }
        // chained sweep: W1 as the B operand plus a ones column (n == lat) for g
        std::vector<double> wbf((size_t)nkb * 32, 0.0);
        for (int kb = 0; kb < nkb; ++kb)
          for (int l = 0; l < 32; ++l) {
            const int k = 4 * kb + (l & 3), n = l >> 2;
            if (k >= h.n_hidden) continue;
            if (n < lat) wbf[(size_t)kb * 32 + l] = h.W1[(size_t)k * lat + n];
            else if (n == lat) wbf[(size_t)kb * 32 + l] = 1.0;
          }
        if ((rc = upload(c, wbf.data(), wbf.size(), const_cast<double**>(&d.wbfrag)))) return rc;
        if ((rc = upload(c, fr.data(), fr.size(), const_cast<double**>(&d.w1frag))) ||
            (rc = upload(c, vr.data(), vr.size(), const_cast<double**>(&d.v_row))) ||
            (rc = upload(c, rw.data(), rw.size(), const_cast<int**>(&d.row_w))))
          return rc;
        hw.k0 = k0;
        hw.w = rw;
        hw.maxw = (int)wmax;
      } else {
        if ((rc = upload(c, ek.data(), ek.size(), const_cast<int**>(&d.ell_k)))) return rc;
      }
    }
  } else {
    if ((rc = upload(c, h.W1, (size_t)h.n_out * lat, const_cast<double**>(&d.W1)))) return rc;
    d.W1t = nullptr;
    d.b1 = nullptr; d.indptr = nullptr; d.indices = nullptr; d.data = nullptr;
    d.scale = nullptr; d.shift = nullptr;
  }
  return 0;
}

// ---- evaluation units (large blocks) --------------------------------------
// A block whose subnet, rows or interface decoder would not fit one CTA's
// shared memory next to a few slots is evaluated as a sequence of units:
//  * row units: a contiguous chunk of the block's sampled rows with the
//    interior subnet restricted to the outputs those rows reference and the
//    interface decoder restricted to the interface outputs they reference
//    (extract_subnet, hyper.py:200-222, applied once more: every kept output
//    is bitwise the full subnet's; test_hyper.py:194-201 pins that invariant);
//    each adds its rows' Gram contribution R^T R, R^T r, r^T r to the block;
//  * constraint units: a chunk of the full interface decoder's outputs and
//    the matching columns of C A_i, adding C A_i g / C A_i J over the chunk
//    (driver.py:371-373).
// Sums over rows / interface outputs are then taken chunk by chunk (unit
// order, deterministic) instead of in one pass: same terms, rounding only.

struct HostDecoder {          // owning copy of a (restricted) decoder
  std::vector<double> W1, b1, data, scale, shift;
  std::vector<int64_t> indptr, indices;
  ddnm_decoder d{};
  void finish() {
    d.n_out = (int32_t)scale.size();
    d.n_hidden = (int32_t)b1.size();
    d.W1 = W1.empty() ? nullptr : W1.data();
    d.b1 = b1.data(); d.indptr = indptr.data(); d.indices = indices.data(); d.data = data.data();
    d.scale = scale.data(); d.shift = shift.data();
    if (d.n_out == 0) { static const double z = 0.0; d.W1 = &z; d.n_hidden = 0; }
  }
};

// the decoder restricted to the outputs `outs` (in that order): hidden units
// are the sorted union of their entries, entries keep storage order
void restrict_decoder(const ddnm_decoder& h, int lat, const std::vector<int>& outs, HostDecoder& r) {
  std::vector<int> hid;
  for (int o : outs)
    for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e) hid.push_back((int)h.indices[e]);
  std::sort(hid.begin(), hid.end());
  hid.erase(std::unique(hid.begin(), hid.end()), hid.end());
  std::map<int, int> pos;
  for (size_t k = 0; k < hid.size(); ++k) pos[hid[k]] = (int)k;
  r.W1.resize(hid.size() * lat);
  r.b1.resize(hid.size());
  for (size_t k = 0; k < hid.size(); ++k) {
    for (int d = 0; d < lat; ++d) r.W1[k * lat + d] = h.W1[(size_t)hid[k] * lat + d];
    r.b1[k] = h.b1[hid[k]];
  }
  r.indptr.assign(1, 0);
  r.indices.clear(); r.data.clear(); r.scale.clear(); r.shift.clear();
  for (int o : outs) {
    for (int64_t e = h.indptr[o]; e < h.indptr[o + 1]; ++e) {
      r.indices.push_back(pos[(int)h.indices[e]]);
      r.data.push_back(h.data[e]);
    }
    r.indptr.push_back((int64_t)r.indices.size());
    r.scale.push_back(h.scale[o]);
    r.shift.push_back(h.shift[o]);
  }
  r.finish();
}

struct HostUnit {
  HostDecoder in, ga;
  std::vector<int64_t> rows, cols, gio;
  std::vector<double> CA;
  std::vector<int> iout_map, gout_map, row_map;
  ddnm_block blk{};
  int flags = 0;
};

struct UnitLimits { int rows, hidden, outs, grefs, gchunk; };

// <= 128 rows / 1536 hidden units per row unit (config 3: 128 units, 4
// slots, 120 ms per 1024 mu; 256 rows: 115 units but only 2 slots fit,
// 140-145 ms; 768-1024 hidden: more units, 129-142 ms; profiles/r2i.log);
// DDNM_UNIT_* override (tests, experiments)
UnitLimits unit_limits() {
  UnitLimits L{128, 1536, 512, 128, 256};
  if (const char* ur = getenv("DDNM_UNIT_ROWS")) L.rows = std::max(1, atoi(ur));
  if (const char* ug = getenv("DDNM_UNIT_GAM")) L.gchunk = std::max(8, atoi(ug));
  if (const char* uh = getenv("DDNM_UNIT_HIDDEN")) L.hidden = std::max(64, atoi(uh));
  if (const char* uo = getenv("DDNM_UNIT_OUTS")) L.outs = std::max(16, atoi(uo));
  return L;
}

// blocks are split when any block is too large for one CTA's shared-memory
// plan (or DDNM_UNIT_ROWS forces it); autoencoder WFPC collocation only
bool wants_units(const ddnm_artifacts* a) {
  bool need = false, nogappy = true;
  for (int b = 0; b < a->n_blocks; ++b) {
    const ddnm_block& k = a->blocks[b];
    if (k.interior.n_hidden > 2048 || k.n_io > 512 || k.n_rows > 256 || k.interface.n_out > 512)
      need = true;
    if (k.n_basis > 0) nogappy = false;
  }
  const bool can = a->map_kind == DDNM_MAP_AUTOENCODER && a->constraint_mode == DDNM_CON_WFPC;
  return (need || getenv("DDNM_UNIT_ROWS")) && can && nogappy && !getenv("DDNM_NO_UNITS");
}

// split block k into units (row chunks, then interface-output chunks)
int split_block(const ddnm_artifacts* a, const ddnm_block& k, const HostRows& hr,
                const UnitLimits& L, std::vector<HostUnit>& out) {
  const int nr = k.n_rows, nio = k.n_io;
  const ddnm_decoder& di = k.interior;
  std::vector<int> omark(std::max(nio, 1), 0), hmark(std::max(di.n_hidden, 1), 0),
      gmark(std::max(k.n_gio, 1), 0);
  int stamp = 0;
  // rows in node order (the u and v rows of a node and the rows of
  // neighbouring nodes reference the same outputs and hidden units)
  const int64_t nn = (int64_t)a->nx * a->ny;
  std::vector<int> order(nr);
  for (int r = 0; r < nr; ++r) order[r] = r;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    const int64_t px = k.res_rows[x] % nn, py = k.res_rows[y] % nn;
    if (px != py) return px < py;
    return k.res_rows[x] < k.res_rows[y];
  });
  int r0 = 0;
  bool first_rows = true;
  auto refs = [&](int r, std::vector<int>& io, std::vector<int>& gi) {
    io.clear(); gi.clear();
    for (int e = 0; e < hr.nent[r]; ++e) {
      const int c = hr.col[(size_t)e * nr + r];
      if (c < nio) io.push_back(c); else gi.push_back(c - nio);
    }
  };
  auto flush = [&](int r1) {
    if (r1 <= r0) return;
    out.emplace_back();
    HostUnit& u = out.back();
    std::vector<int> io, gi, uo, ug;
    for (int q = r0; q < r1; ++q) {
      refs(order[q], io, gi);
      uo.insert(uo.end(), io.begin(), io.end());
      ug.insert(ug.end(), gi.begin(), gi.end());
    }
    std::sort(uo.begin(), uo.end()); uo.erase(std::unique(uo.begin(), uo.end()), uo.end());
    std::sort(ug.begin(), ug.end()); ug.erase(std::unique(ug.begin(), ug.end()), ug.end());
    restrict_decoder(k.interior, k.n_int, uo, u.in);
    std::vector<int> gouts;
    for (int g : ug) gouts.push_back((int)k.gio[g]);
    restrict_decoder(k.interface, k.n_gam, gouts, u.ga);
    for (int q = r0; q < r1; ++q) {
      u.rows.push_back(k.res_rows[order[q]]);
      u.row_map.push_back(order[q]);
    }
    for (int o : uo) u.cols.push_back(k.cols[o]);
    for (int g : ug) u.cols.push_back(k.cols[nio + g]);
    for (size_t g = 0; g < ug.size(); ++g) u.gio.push_back((int64_t)g);
    u.iout_map = uo;
    u.flags = UF_ROWS | (first_rows ? 0 : UF_ACC_GRAM);
    first_rows = false;
    r0 = r1;
  };
  int n_o = 0, n_h = 0, n_g = 0;
  ++stamp;
  std::vector<int> io, gi;
  for (int q = 0; q < nr; ++q) {
    const int r = order[q];
    refs(r, io, gi);
    // what this row would add to the current unit
    int add_o = 0, add_h = 0, add_g = 0;
    const int st2 = stamp + 1;
    std::vector<int> newh;
    for (int o : io) {
      if (omark[o] == stamp || omark[o] == st2) continue;
      omark[o] = st2; ++add_o;
      for (int64_t e = di.indptr[o]; e < di.indptr[o + 1]; ++e) {
        const int h = (int)di.indices[e];
        if (hmark[h] == stamp || hmark[h] == st2) continue;
        hmark[h] = st2; ++add_h; newh.push_back(h);
      }
    }
    for (int g : gi) if (gmark[g] != stamp && gmark[g] != st2) { gmark[g] = st2; ++add_g; }
    const bool over = q > r0 && (q - r0 + 1 > L.rows || n_o + add_o > L.outs ||
                                 n_h + add_h > L.hidden || n_g + add_g > L.grefs);
    if (over) {
      flush(q);
      stamp += 2;
      n_o = n_h = n_g = 0;
      --q;          // re-add this row to the fresh unit
      continue;
    }
    // commit the row
    for (int o : io) if (omark[o] == st2) omark[o] = stamp;
    for (int h : newh) hmark[h] = stamp;
    for (int g : gi) if (gmark[g] == st2) gmark[g] = stamp;
    n_o += add_o; n_h += add_h; n_g += add_g;
  }
  flush(nr);
  // constraint units: chunks of the full interface decoder (WFPC)
  const int ngo = k.interface.n_out;
  bool first_con = true;
  for (int o0 = 0; o0 < ngo; o0 += L.gchunk) {
    const int o1 = std::min(ngo, o0 + L.gchunk);
    out.emplace_back();
    HostUnit& u = out.back();
    std::vector<int> gouts;
    for (int o = o0; o < o1; ++o) gouts.push_back(o);
    restrict_decoder(k.interface, k.n_gam, gouts, u.ga);
    std::vector<int> none;
    restrict_decoder(k.interior, k.n_int, none, u.in);
    u.gout_map = gouts;
    u.CA.resize((size_t)a->n_c * (o1 - o0));
    for (int c = 0; c < a->n_c; ++c)
      for (int o = o0; o < o1; ++o) u.CA[(size_t)c * (o1 - o0) + (o - o0)] = k.CA[(size_t)c * ngo + o];
    u.flags = UF_CON | (first_con ? 0 : UF_ACC_CON);
    first_con = false;
  }
  for (HostUnit& u : out) {
    ddnm_block& b = u.blk;
    b.n_int = k.n_int; b.n_gam = k.n_gam;
    b.interior = u.in.d; b.interface = u.ga.d;
    b.n_rows = (int32_t)u.rows.size();
    b.res_rows = u.rows.empty() ? nullptr : u.rows.data();
    b.n_cols = (int32_t)u.cols.size();
    b.cols = u.cols.empty() ? nullptr : u.cols.data();
    b.n_io = u.in.d.n_out;
    b.n_gio = (int32_t)u.gio.size();
    b.gio = u.gio.empty() ? nullptr : u.gio.data();
    b.CA = u.CA.empty() ? nullptr : u.CA.data();
    b.n_basis = 0; b.weights = nullptr;
  }
  return 0;
}

int64_t nnz_of(const ddnm_decoder& d, int kind) {
  return kind == DDNM_MAP_AUTOENCODER ? d.indptr[d.n_out] : 0;
}

}  // namespace

extern "C" {

const char* ddnm_last_error(void) { return g_err.c_str(); }
int ddnm_abi_version(void) { return DDNM_ABI_VERSION; }

int ddnm_ctx_create(int32_t device, const ddnm_artifacts* a, int32_t slots, ddnm_ctx** out) {
  if (!a || !out) return fail(DDNM_EINVAL, "null argument");
  *out = nullptr;
  if (a->abi_version != DDNM_ABI_VERSION) return fail(DDNM_EINVAL, "ABI version mismatch");
  if (a->n_blocks < 1 || a->n_blocks > MAXB) return fail(DDNM_EINVAL, "need 1..16 blocks");
  if (a->n_c < 1) return fail(DDNM_EINVAL, "multiplier dimension must be positive");
  if (a->nx < 2 || a->ny < 2 || !(a->nu > 0)) return fail(DDNM_EINVAL, "bad grid");
  if (a->map_kind != DDNM_MAP_AUTOENCODER && a->map_kind != DDNM_MAP_LINEAR)
    return fail(DDNM_EINVAL, "unknown map kind");
  if (a->constraint_mode != DDNM_CON_WFPC && a->constraint_mode != DDNM_CON_SRPC)
    return fail(DDNM_EINVAL, "unknown constraint mode");
  const int ni = a->blocks[0].n_int, ng = a->blocks[0].n_gam;
  for (int b = 0; b < a->n_blocks; ++b) {
    const ddnm_block& k = a->blocks[b];
    if (k.n_int != ni || k.n_gam != ng)
      return fail(DDNM_EUNSUPPORTED, "blocks with different latent dims are not compiled");
    if (k.interior.n_out != k.n_io) return fail(DDNM_EINVAL, "interior decoder outputs != n_io");
    if (k.n_cols != k.n_io + k.n_gio) return fail(DDNM_EINVAL, "n_cols != n_io + n_gio");
    if (k.n_rows < 1) return fail(DDNM_EINVAL, "sample row set is empty");
    if (!k.CA) return fail(DDNM_EINVAL, "missing CA");
    int rc;
    if ((rc = check_decoder(k.interior, ni, a->map_kind, "interior"))) return rc;
    if ((rc = check_decoder(k.interface, ng, a->map_kind, "interface"))) return rc;
    for (int g = 0; g < k.n_gio; ++g)
      if (k.gio[g] < 0 || k.gio[g] >= k.interface.n_out) return fail(DDNM_EINVAL, "gio out of range");
    if (a->constraint_mode == DDNM_CON_SRPC && k.interface.n_out != k.n_gio)
      return fail(DDNM_EINVAL, "SRPC interface decoder must be restricted to the gio outputs");
    if (k.n_basis < 0 || k.n_basis > k.n_rows || (k.n_basis > 0 && !k.weights))
      return fail(DDNM_EINVAL, "gappy weights need 1..n_rows basis vectors");
  }
  auto* c = new ddnm_ctx();
  int rc = 0;
  auto bail = [&](int r) {
    ddnm_ctx_destroy(c);
    return r;
  };
  if (device < 0) {
    if (cudaGetDevice(&device) != cudaSuccess) return bail(fail(DDNM_ECUDA, "no CUDA device"));
  }
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(DDNM_ECUDA, "cudaSetDevice failed"));
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "cudaGetDeviceProperties failed"));
  if (prop.major != 10) return bail(fail(DDNM_EUNSUPPORTED, "libddnm is built for sm_100a (B200)"));
  c->sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "stream create failed"));

  Params& P = c->P;
  std::memset(&P, 0, sizeof(P));
  P.nb = a->n_blocks;
  P.n_C = a->n_c;
  P.map_kind = a->map_kind;
  c->map_kind = a->map_kind;
  P.con_mode = a->constraint_mode;
  P.act = a->activation;
  P.nx = a->nx;
  P.ny = a->ny;
  P.nu = a->nu;
  P.hx = 2.0 / (a->nx + 1);
  P.hy = 0.05 / (a->ny + 1);
  const int W = ni + ng;
  int xoff = 0, row_off = 0, iout = 0, gout = 0, Roff = 0, cjoff = 0, ijoff = 0, gjoff = 0, eboff = 0;
  int max_nh = 0, max_io = 0, max_gam = 0, max_rows = 0, max_nbz = 0, out_off = 0, outR_off = 0;
  std::vector<HostWindows> hwin(2 * a->n_blocks);
  // device tables of one block (or evaluation unit): decoders, stencil rows,
  // gio, constraint matrix, gappy weights
  auto setup = [&](const ddnm_block& k, BlockDev& B, HostWindows* hw2, HostRows& hr) -> int {
    int rc2;
    HostWindows tmp[2];
    B.ni = ni; B.ng = ng; B.w = W;
    B.nrows = k.n_rows; B.n_io = k.n_io; B.n_gio = k.n_gio;
    B.uflags = UF_ROWS | UF_CON;
    B.iout_map = nullptr; B.gout_map = nullptr; B.row_map = nullptr;
    if ((rc2 = upload_decoder(c, k.interior, ni, a->map_kind, a->activation, B.in, hw2 ? hw2[0] : tmp[0])))
      return rc2;
    if ((rc2 = upload_decoder(c, k.interface, ng, a->map_kind, a->gam_activation, B.ga,
                              hw2 ? hw2[1] : tmp[1])))
      return rc2;
    if ((rc2 = build_stencil(a, k, hr))) return rc2;
    StRows& R = B.rows;
    if ((rc = upload(c, hr.gu.data(), hr.gu.size(), const_cast<int**>(&R.gu))) ||
        (rc = upload(c, hr.gv.data(), hr.gv.size(), const_cast<int**>(&R.gv))) ||
        (rc = upload(c, hr.nent.data(), hr.nent.size(), const_cast<int**>(&R.nent))) ||
        (rc = upload(c, hr.bflags.data(), hr.bflags.size(), const_cast<int**>(&R.bflags))) ||
        (rc = upload(c, hr.col.data(), hr.col.size(), const_cast<int**>(&R.col))) ||
        (rc = upload(c, hr.src.data(), hr.src.size(), const_cast<int**>(&R.src))) ||
        (rc = upload(c, hr.sgu.data(), hr.sgu.size(), const_cast<int**>(&R.src_gu))) ||
        (rc = upload(c, hr.sgv.data(), hr.sgv.size(), const_cast<int**>(&R.src_gv))) ||
        (rc = upload(c, hr.bxc.data(), hr.bxc.size(), const_cast<double**>(&R.bxc))) ||
        (rc = upload(c, hr.byc.data(), hr.byc.size(), const_cast<double**>(&R.byc))) ||
        (rc = upload(c, hr.cdc.data(), hr.cdc.size(), const_cast<double**>(&R.cdc))) ||
        (rc = upload(c, hr.xc.data(), hr.xc.size(), const_cast<double**>(&R.xc))) ||
        (rc = upload(c, hr.yc.data(), hr.yc.size(), const_cast<double**>(&R.yc))))
      return rc;
    if ((rc = upload_i32(c, k.gio, (size_t)k.n_gio, const_cast<int**>(&B.gio)))) return rc;
    const size_t ca_cols = a->constraint_mode == DDNM_CON_SRPC ? (size_t)ng : (size_t)k.interface.n_out;
    B.CA = nullptr;
    if (k.CA && (rc = upload(c, k.CA, (size_t)P.n_C * ca_cols, const_cast<double**>(&B.CA)))) return rc;
    B.nbz = k.n_basis;
    B.wts = nullptr;
    if (k.n_basis > 0 &&
        (rc = upload(c, k.weights, (size_t)k.n_basis * k.n_rows, const_cast<double**>(&B.wts))))
      return rc;
    return 0;
  };
  std::vector<HostRows> hrows(a->n_blocks);
  for (int b = 0; b < P.nb; ++b) {
    const ddnm_block& k = a->blocks[b];
    BlockDev& B = P.blk[b];
    if ((rc = setup(k, B, &hwin[2 * b], hrows[b]))) return bail(rc);
    B.real = b;
    B.xoff = xoff; B.row_off = row_off; B.iout_off = iout; B.gout_off = gout; B.R_off = Roff;
    B.cjac_off = cjoff; B.intJ_off = ijoff; B.gamJ_off = gjoff; B.eb_off = eboff;
    B.out_off = out_off;
    B.outR_off = outR_off;
    out_off += k.n_basis > 0 ? k.n_basis : k.n_rows;
    outR_off += (k.n_basis > 0 ? k.n_basis : k.n_rows) * W;
    max_nbz = std::max(max_nbz, (int)k.n_basis);
    xoff += W; row_off += k.n_rows; iout += k.n_io; gout += k.interface.n_out;
    Roff += k.n_rows * W; cjoff += P.n_C * ng; ijoff += k.n_io * ni; gjoff += k.interface.n_out * ng;
    eboff += W * (W + 1) / 2 + W + P.n_C + P.n_C * ng + 1;
    max_nh = std::max(max_nh, B.in.n_hidden + B.ga.n_hidden);
    max_io = std::max(max_io, k.n_io);
    max_gam = std::max(max_gam, k.interface.n_out);
    max_rows = std::max(max_rows, k.n_rows);
  }
  // evaluation units for blocks too large for one CTA (configs 3/4): every
  // block becomes units when any block needs splitting (DDNM_UNIT_ROWS forces
  // it, for tests on small instances)
  {
    const UnitLimits L = unit_limits();
    if (wants_units(a)) {
      std::vector<BlockDev> units;
      max_nh = max_io = max_gam = max_rows = 0;
      for (int b = 0; b < P.nb; ++b) {
        const ddnm_block& k = a->blocks[b];
        const BlockDev& RB = P.blk[b];
        P.u_bnd[b] = (int)units.size();
        std::vector<HostUnit> hu;
        if ((rc = split_block(a, k, hrows[b], L, hu))) return bail(rc);
        for (HostUnit& u : hu) {
          BlockDev U;
          std::memset(&U, 0, sizeof U);
          HostRows uhr;
          if ((rc = setup(u.blk, U, nullptr, uhr))) return bail(rc);
          U.uflags = u.flags;
          U.real = b;
          U.xoff = RB.xoff; U.eb_off = RB.eb_off; U.cjac_off = RB.cjac_off;
          U.iout_off = RB.iout_off; U.intJ_off = RB.intJ_off;
          U.gout_off = RB.gout_off; U.gamJ_off = RB.gamJ_off;
          U.row_off = RB.row_off;
          U.out_off = RB.out_off;
          U.outR_off = RB.outR_off;
          U.R_off = RB.R_off;
          if (!u.row_map.empty() &&
              (rc = upload(c, u.row_map.data(), u.row_map.size(), const_cast<int**>(&U.row_map))))
            return bail(rc);
          if (!u.iout_map.empty() &&
              (rc = upload(c, u.iout_map.data(), u.iout_map.size(), const_cast<int**>(&U.iout_map))))
            return bail(rc);
          if (!u.gout_map.empty() &&
              (rc = upload(c, u.gout_map.data(), u.gout_map.size(), const_cast<int**>(&U.gout_map))))
            return bail(rc);
          max_nh = std::max(max_nh, U.in.n_hidden + U.ga.n_hidden);
          max_io = std::max(max_io, U.in.n_out);
          max_gam = std::max(max_gam, U.ga.n_out);
          max_rows = std::max(max_rows, U.nrows);
          units.push_back(U);
        }
      }
      P.u_bnd[P.nb] = (int)units.size();
      P.n_units = (int)units.size();
      if ((rc = upload(c, units.data(), units.size(), const_cast<BlockDev**>(&P.units)))) return bail(rc);
      c->n_units = P.n_units;
    }
  }
  P.n_D = xoff;
  P.nK = P.n_D + P.n_C;
  P.b_lo = 0;
  P.b_hi = P.nb;
  // block-structured KKT for block systems W + n_C <= 32 always; up to 96 for
  // autoencoder ROMs (dd16: 478 -> 92 ms per 1024 mu).  The LS-ROMs' block
  // factorisations lose pivots to multiplier rows at nearly every solve
  // (c0_ls: 138 -> 150 ms with the attempt), so they go straight to the
  // dense LU there.  DDNM_KKT_BLOCK_MAX overrides.
  P.kkt_block_max = a->map_kind == DDNM_MAP_AUTOENCODER ? 96 : 32;
  // hidden pre-activation: per-unit DFMA (default) or FP64 tensor-core tiles
  // (DDNM_HIDDEN_DMMA=1, hidden_range).  Measured (profiles/r2e_hidden_ab.log):
  // the tiles are 3-5% slower at config 2 (36.1 vs 34.4-35.1 ms per 4096 mu)
  // and 11% at config 3 (156.6 vs 140.1 ms per 1024 mu, 2 slots: the B
  // operand's 8 slot columns hold 2): the pre-activation is ~1/4 of the
  // phase's FP64 work (the activations dominate) and the tiles add a
  // shared-memory round trip of Z between the mma chains and the activations.
  P.hid_dmma = getenv("DDNM_HIDDEN_DMMA") ? 1 : 0;
  if (const char* kb = getenv("DDNM_KKT_BLOCK_MAX")) P.kkt_block_max = std::min(96, atoi(kb));
  P.total_rows = row_off;
  P.tot_iout = iout; P.tot_gout = gout; P.tot_R = Roff; P.tot_cjac = cjoff;
  P.tot_intJ = ijoff; P.tot_gamJ = gjoff;
  P.tot_out = out_off; P.tot_outR = outR_off;
  c->n_D = P.n_D; c->n_C = P.n_C; c->nb = P.nb;
  c->tot_rows = row_off; c->tot_iout = iout; c->tot_gout = gout; c->tot_R = Roff;
  c->tot_cjac = cjoff; c->tot_intJ = ijoff; c->tot_gamJ = gjoff;
  // RBF
  const ddnm_rbf& r = a->rbf;
  P.rbf_P = r.n_centers; P.rbf_R = r.n_mono;
  if (r.n_centers > 0) {
    if ((rc = upload(c, r.y, (size_t)r.n_centers * 2, const_cast<double**>(&P.rbf_y)))) return bail(rc);
    if ((rc = upload(c, r.coeffs, (size_t)(r.n_centers + r.n_mono) * P.n_D,
                     const_cast<double**>(&P.rbf_coeffs)))) return bail(rc);
    if ((rc = upload_i32(c, r.powers, (size_t)r.n_mono * 2, const_cast<int**>(&P.rbf_pow)))) return bail(rc);
    for (int k = 0; k < 2; ++k) {
      P.rbf_shift[k] = r.shift[k]; P.rbf_scale[k] = r.scale[k];
      P.rbf_lo[k] = r.lo[k]; P.rbf_hi[k] = r.hi[k];
    }
    P.rbf_eps = r.epsilon;
  }
  // shared-memory plan (doubles)
  const bool ae = a->map_kind == DDNM_MAP_AUTOENCODER;
  // per-slot scratch plan; the interior Jacobian rows stay in shared memory
  // when they fit, otherwise they go to a per-slot L2 scratch (gJ)
  // level 0: both Jacobian row sets in shared memory; 1: interface rows in L2;
  // 2: both in L2 (per-slot global scratch)
  auto plan_scratch = [&](int level) {
    int scr = 0;
    P.scr_sig = scr; scr += ae ? max_nh + 32 : 0;    // +32: zero padding read past
    P.scr_dsig = scr; scr += ae ? max_nh + 32 : 0;   // n_hidden by the sweeps
    P.scr_gint = scr; scr += max_io;
    if (ae && level < 2) { P.scr_jint = scr; scr += max_io * ni; } else { P.scr_jint = -1; }
    P.scr_ggam = scr; scr += max_gam;
    if (ae && level < 1) { P.scr_jgam = scr; scr += max_gam * ng; } else { P.scr_jgam = -1; }
    // R and r are produced after the sweep has consumed sigma/sigma': alias them
    if (ae && max_rows * (W + 1) <= 2 * max_nh) {
      P.scr_R = P.scr_sig;
      P.scr_r = P.scr_sig + max_rows * W;
    } else {
      P.scr_R = scr; scr += max_rows * W;
      P.scr_r = scr; scr += max_rows;
    }
    P.scr_RB = -1;
    if (max_nbz > 0) { P.scr_RB = scr; scr += max_nbz * (W + 1); }
    return scr;
  };
  int scr = plan_scratch(0);
  P.gJ_stride = ae ? max_io * ni : 0;
  P.gJg_stride = ae ? max_gam * ng : 0;
  const int kkt_need = std::max(P.nK * (P.nK + 1) + 6 * P.nK,
                                P.nb * (W + P.n_C) * (W + P.n_C + 1) + P.nb * W +
                                    P.n_C * (P.n_C + 1) + P.n_C + P.nb * P.n_C + 4 * P.nK);
  const int ls_need = P.nb * ng * P.n_C + P.nb * ng;
  const int rbf_need = r.n_centers + r.n_mono;
  P.scr_size = std::max(std::max(scr, kkt_need), std::max(ls_need, rbf_need));
  P.scr_size = (P.scr_size + 1) & ~1;
  P.eb_size = eboff + P.n_D + P.n_C + 2;
  P.eb_rho = eboff; P.eb_con = eboff + P.n_D; P.eb_scal = eboff + P.n_D + P.n_C;
  P.eb_size = (P.eb_size + 1) & ~1;
  const int state_d = (int)((sizeof(SlotState) + 7) / 8);
  // pick G (slots per CTA): the largest compiled G whose footprint fits,
  // preferring the interior Jacobian rows in shared memory
  const size_t smem_cap = (size_t)prop.sharedMemPerBlockOptin - 1024;
  const int rbf_need2 = rbf_need;
  // kg: the KKT workspace lives in a per-slot global scratch (kernels
  // instantiated with KG = true), so it does not count against shared memory
  auto scr_total = [&](int level, bool kg = false) {
    int s0 = plan_scratch(level);
    // (kg: the Schur block, n_C x (n_C + 1), stays in this scratch)
    int t = std::max(std::max(s0, kg ? P.n_C * (P.n_C + 1) : kkt_need), std::max(ls_need, rbf_need2));
    return (t + 1) & ~1;
  };
  // ebg: the evaluation buffers live in global memory (Params::eb_glob)
  auto footprint = [&](int G, int level, bool kg = false, bool ebg = false) {
    return ((size_t)state_d * G +
            (size_t)G * (8 * P.nK + (ebg ? 0 : 2 * P.eb_size) + scr_total(level, kg))) * 8;
  };
  bool kern_ebg = false;
  const Kernels* kern = nullptr;
  int kern_level = 0;
  const char* jl = getenv("DDNM_JLEVEL");
  const int lvl_lo = jl ? atoi(jl) : 0, lvl_hi = jl ? atoi(jl) : (ae ? 2 : 0);
  // planner (see below: even G first, then the largest; measured at
  // config 0 with the tensor-core Gram: 4 slots with the Jacobian rows in L2
  // 35.7-37.1 ms per 4096 mu, vs 41.5 ms for 2 slots with them in shared memory)
  // kernels with the KKT workspace in global memory only when nothing else fits.
  // Slot count: the largest G that fits, even G first (odd G takes the
  // slower reduce-scatter path of the decoder sweep: c0_nmg 45.1 ms at 2
  // slots vs 47.7 ms at 3).  Level: for that G, the lowest Jacobian-row level
  // whose footprint stays under a soft cap of 192 KB (>= ~36 KB of L1 left),
  // else the lowest level that fits: at config 3's layout (c3s, 120^2, 1024
  // mu) 2 slots with the rows in shared memory (205 KB) take 33.3 ms and with
  // them in L2 (146 KB) 29.9 ms; c0_srpc keeps 2 slots at 219 KB (216 ms vs
  // 243 ms for 1 slot).  DDNM_SMEM_SOFT_CAP overrides (bytes).
  // (200 KB: config 3's evaluation units at 4 slots need 199 KB and take
  // 120 ms per 1024 mu vs 140 ms at 2 slots; config 4 at 4 slots needs 214 KB
  // and is slower than at 2, profiles/r2i.log)
  size_t soft_cap = std::min<size_t>(smem_cap, 200 * 1024);
  if (const char* sc = getenv("DDNM_SMEM_SOFT_CAP")) soft_cap = std::min<size_t>(smem_cap, (size_t)atoll(sc));
  // ranking: a footprint under the soft cap first (the L1 left for the
  // weights matters more than one more slot: config 4 with the evaluation
  // buffers in L2 takes 501 ms per 256 mu at 2 slots / 193 KB and 725 ms at
  // 4 slots / 214 KB, profiles/r2h.log), then even before odd, then larger
  auto better = [](int g, bool soft, int best, bool best_soft) {
    if (best < 0) return true;
    if (soft != best_soft) return soft;
    if ((g % 2 == 0) != (best % 2 == 0)) return g % 2 == 0;
    return g > best;
  };
  bool kern_soft = false;
  // pass 0: everything in shared memory; pass 1: the KKT workspace in L2
  // (KG kernels), and -- when that alone leaves slots on the table -- the
  // evaluation buffers too (config 4: 2 x 5.8k doubles per slot)
  // only for instances split into evaluation units: their rounds are long
  // enough to hide the buffers' L2 traffic (config 4: 501 ms at 2 slots vs
  // 544-573 ms at 1 slot with the buffers in shared memory); dd16's small
  // blocks are not (27.6 ms at 1 slot in shared memory, 58 ms at 4 slots
  // with the buffers in L2, profiles/r2k_bench.json)
  const bool ebg_ok = P.units && !getenv("DDNM_NO_EB_GLOBAL");
  for (int pass = 0; pass < 2 && !kern; ++pass) {
    for (const auto& k : kernel_table()) {
      if (k.ni != ni || k.ng != ng || k.kkt_global != (pass == 1)) continue;
      if (slots > 0 && k.g != slots) continue;
      for (int eg = 0; eg < (pass == 1 && ebg_ok ? 2 : 1); ++eg) {
        int lv = -1;
        bool soft = false;
        for (int level = lvl_lo; level <= lvl_hi && lv < 0; ++level)
          if (footprint(k.g, level, k.kkt_global, eg) <= soft_cap) { lv = level; soft = true; }
        for (int level = lvl_lo; level <= lvl_hi && lv < 0; ++level)
          if (footprint(k.g, level, k.kkt_global, eg) <= smem_cap) lv = level;
        if (lv < 0) continue;
        if (better(k.g, soft, kern ? kern->g : -1, kern_soft)) {
          kern = &k; kern_level = lv; kern_ebg = eg; kern_soft = soft;
        }
        if (soft) break;   // buffers in shared memory when they fit this G under the cap
      }
    }
  }
  if (!kern) {
    char buf[160];
    snprintf(buf, sizeof buf,
             "no compiled kernel for n_int=%d n_gam=%d slots=%d fitting %zu B smem "
             "(declare the pair in csrc/latent_dims.txt or DDNM_LATENT_DIMS and rebuild)",
             ni, ng, slots, smem_cap);
    return bail(fail(DDNM_EUNSUPPORTED, buf));
  }
  P.scr_size = scr_total(kern_level, kern->kkt_global);
  c->K = *kern;
  c->kkt_stride = kern->kkt_global ? (size_t)((kkt_need + 31) & ~31) : 0;
  P.kkt_stride = (long long)c->kkt_stride;
  // tiles of consecutive outputs for the tensor-core sweep (P = 8 / G outputs each)
  if (getenv("DDNM_DMMA") && ae && 8 % kern->g == 0 && !P.units) {
    const int Pt = 8 / kern->g;
    for (int b = 0; b < P.nb; ++b) {
      if (hwin[2 * b].k0.empty() || hwin[2 * b + 1].k0.empty()) continue;
      std::vector<TileRec> tiles;
      int n_in = 0;
      for (int which = 0; which < 2; ++which) {
        if (which == 1) n_in = (int)tiles.size();
        const HostWindows& hw = hwin[2 * b + which];
        const int n = (int)hw.k0.size();
        int o = 0;
        while (o < n) {
          int lo = hw.k0[o], hi = hw.k0[o] + hw.w[o];
          int cnt = 1;
          while (cnt < Pt && o + cnt < n) {
            const int nlo = std::min(lo, hw.k0[o + cnt]);
            const int nhi = std::max(hi, hw.k0[o + cnt] + hw.w[o + cnt]);
            if (nhi - nlo > hw.maxw + Pt + 3) break;
            lo = nlo; hi = nhi; ++cnt;
          }
          TileRec t;
          std::memset(&t, 0, sizeof t);
          t.o0 = o; t.cnt = cnt | (which << 8); t.kb_lo = lo / 4; t.kb_hi = (hi - 1) / 4;
          for (int j = 0; j < cnt; ++j) { t.k0[j] = hw.k0[o + j]; t.w[j] = hw.w[o + j]; }
          if (t.kb_hi - t.kb_lo + 1 > 10) return bail(fail(DDNM_EUNSUPPORTED, "sweep tile wider than 10 k-blocks"));
          tiles.push_back(t);
          o += cnt;
        }
      }
      // B-operand W2 values per tile in fragment order (mu-independent)
      std::vector<double> tv(tiles.size() * 10 * 32, 0.0);
      const int Gk = kern->g;
      for (size_t t = 0; t < tiles.size(); ++t) {
        const TileRec& T = tiles[t];
        const int which = T.cnt >> 8, cnt = T.cnt & 0xff;
        const ddnm_decoder& h = which == 0 ? a->blocks[b].interior : a->blocks[b].interface;
        for (int i = 0; i <= T.kb_hi - T.kb_lo; ++i)
          for (int l = 0; l < 32; ++l) {
            const int tig = l & 3, oo = (l >> 2) / Gk;
            if (oo >= cnt) continue;
            const int o = T.o0 + oo;
            const int e = 4 * (T.kb_lo + i) + tig - T.k0[oo];
            if (e >= 0 && e < T.w[oo]) tv[(t * 10 + i) * 32 + l] = h.data[h.indptr[o] + e];
          }
      }
      if ((rc = upload(c, tiles.data(), tiles.size(), const_cast<TileRec**>(&P.blk[b].tiles))) ||
          (rc = upload(c, tv.data(), tv.size(), const_cast<double**>(&P.blk[b].tile_v))))
        return bail(rc);
      P.blk[b].n_tiles = (int)tiles.size();
      P.blk[b].n_tiles_in = n_in;
    }
  }
  if (const char* th = getenv("DDNM_THREADS")) c->threads = std::max(128, std::min(512, atoi(th) / 32 * 32));
  // chained tensor-core sweep (sweep_chain, opt-in with DDNM_SWEEP=1) for
  // banded decoders with latent dims <= 7: tiles of 8 outputs, their banded W2
  // blocks as A fragments, chains of consecutive tiles balanced over the
  // CTA's warps.  Measured at config 0 (4096 mu): 45.8 ms vs 36.5 ms for the
  // per-output sweep -- the HR subnets' outputs are clustered, not contiguous
  // (tile spans 13 k-blocks for 8 outputs of 24 entries: 46% dense A), and
  // the A fragments (230 KB per block) stream from L2 every round.
  const char* swv = getenv("DDNM_SWEEP");
  // DDNM_SWEEP=2: chains for the interface decoder only
  if (ae && ni <= 7 && ng <= 7 && swv && (atoi(swv) == 1 || atoi(swv) == 2) && !getenv("DDNM_DMMA") && !P.units) {
    constexpr int R = 4;
    const bool gam_only = atoi(swv) == 2;
    const int nw = gam_only ? 4 : c->threads / 32;
    for (int b = 0; b < P.nb; ++b) {
      if (hwin[2 * b].k0.empty() || hwin[2 * b + 1].k0.empty()) continue;
      std::vector<TileV2> tl;
      std::vector<int> which_of;
      std::vector<double> afr;
      for (int which = gam_only ? 1 : 0; which < 2; ++which) {
        const HostWindows& hw = hwin[2 * b + which];
        const ddnm_decoder& h = which == 0 ? a->blocks[b].interior : a->blocks[b].interface;
        const int n = (int)hw.k0.size();
        for (int o0 = 0; o0 < n; o0 += 8) {
          TileV2 t;
          t.o0 = o0;
          t.cnt = std::min(8, n - o0);
          t.lo = 0x7fffffff;
          t.hi = -1;
          for (int j = 0; j < t.cnt; ++j) {
            const int o = o0 + j;
            if (hw.w[o] <= 0) continue;
            t.lo = std::min(t.lo, hw.k0[o] / 4);
            t.hi = std::max(t.hi, (hw.k0[o] + hw.w[o] - 1) / 4);
          }
          if (t.hi < 0) t.lo = t.hi = 0;   // rows without entries: g = shift, J = 0
          t.aoff = (int)(afr.size() / 32);
          for (int kb = t.lo; kb <= t.hi; ++kb)
            for (int l = 0; l < 32; ++l) {
              const int j = l >> 2, k = 4 * kb + (l & 3);
              double v = 0.0;
              if (j < t.cnt) {
                const int o = o0 + j, e = k - hw.k0[o];
                if (e >= 0 && e < hw.w[o]) v = h.data[h.indptr[o] + e];
              }
              afr.push_back(v);
            }
          tl.push_back(t);
          which_of.push_back(which);
        }
      }
      long long total = 0;
      for (const auto& t : tl) total += t.hi - t.lo + 1;
      // about two chains per warp, then longest-first assignment to warps
      const long long target = std::max<long long>(1, (total + 2 * nw - 1) / (2 * nw));
      std::vector<ChainRec> ch;
      std::vector<StepRec> steps;
      for (int t = 0; t < (int)tl.size();) {
        ChainRec cr;
        cr.which = which_of[t]; cr.t0 = t; cr.nt = 0;
        int kb0 = 0x7fffffff, kb1 = -1;
        long long cost = 0;
        while (t < (int)tl.size() && which_of[t] == cr.which && cost < target) {
          if (cr.nt >= R && tl[t].lo <= tl[t - R].hi) break;   // ring of R live tiles
          kb0 = std::min(kb0, tl[t].lo);
          kb1 = std::max(kb1, tl[t].hi);
          cost += tl[t].hi - tl[t].lo + 1;
          ++cr.nt;
          ++t;
        }
        // the walk: slot r holds chain tiles r, r + R, ... in turn
        cr.s0 = (int)steps.size();
        int jr[R];
        for (int r = 0; r < R; ++r) jr[r] = r;
        for (int kb = kb0; kb <= kb1; ++kb) {
          StepRec st;
          st.kb = kb; st.last = 0;
          bool any = false;
          for (int r = 0; r < R; ++r) {
            st.aidx[r] = -1;
            if (jr[r] >= cr.nt) continue;
            const TileV2& T = tl[cr.t0 + jr[r]];
            if (kb < T.lo || kb > T.hi) continue;
            st.aidx[r] = T.aoff + kb - T.lo;
            any = true;
            if (kb == T.hi) { st.last |= 1 << r; jr[r] += R; }
          }
          if (any) steps.push_back(st);
        }
        cr.ns = (int)steps.size() - cr.s0;
        ch.push_back(cr);
      }
      // balance: chain cost = its mma count plus a per-step overhead; warp w
      // runs chains w, w + nw, ... of the reordered list (empty chains pad)
      {
        std::vector<long long> cost(ch.size(), 0);
        for (size_t k = 0; k < ch.size(); ++k) {
          for (int i = 0; i < ch[k].ns; ++i)
            for (int r = 0; r < R; ++r) cost[k] += steps[ch[k].s0 + i].aidx[r] >= 0 ? 4 : 0;
          cost[k] += 3 * ch[k].ns;
        }
        std::vector<size_t> order(ch.size());
        for (size_t k = 0; k < order.size(); ++k) order[k] = k;
        std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return cost[x] > cost[y]; });
        std::vector<long long> load(nw, 0);
        std::vector<std::vector<size_t>> per(nw);
        for (size_t k : order) {
          const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
          load[w] += cost[k];
          per[w].push_back(k);
        }
        size_t depth = 0;
        for (const auto& v : per) depth = std::max(depth, v.size());
        std::vector<ChainRec> out(depth * nw);
        for (size_t d = 0; d < depth; ++d)
          for (int w = 0; w < nw; ++w) {
            ChainRec e;
            e.which = 0; e.t0 = 0; e.nt = 0; e.s0 = 0; e.ns = 0;
            out[d * nw + w] = d < per[w].size() ? ch[per[w][d]] : e;
          }
        ch.swap(out);
      }
      BlockDev& BD = P.blk[b];
      if ((rc = upload(c, tl.data(), tl.size(), const_cast<TileV2**>(&BD.t2))) ||
          (rc = upload(c, afr.data(), afr.size(), const_cast<double**>(&BD.afr))) ||
          (rc = upload(c, steps.data(), steps.size(), const_cast<StepRec**>(&BD.steps))) ||
          (rc = upload(c, ch.data(), ch.size(), const_cast<ChainRec**>(&BD.chains))))
        return bail(rc);
      BD.n_chains = (int)ch.size();
      BD.chain_gam_only = gam_only ? 1 : 0;
    }
  }
  P.G = kern->g;
  P.sm_state = 0;
  P.sm_vec = state_d * P.G;
  P.sm_eb = P.sm_vec + P.G * 8 * P.nK;
  P.sm_scr = P.sm_eb + (kern_ebg ? 0 : P.G * 2 * P.eb_size);
  c->ebg = kern_ebg;
  c->smem = footprint(P.G, kern_level, kern->kkt_global, kern_ebg);
  if (!kern->kkt_global && !kern_ebg) {
    const int block_need = P.nb * (W + P.n_C) * (W + P.n_C + 1) + P.nb * W + P.n_C * (P.n_C + 1) +
                           P.n_C + P.nb * P.n_C + 4 * P.nK;
    c->step_scr = (std::max(std::max(block_need, ls_need), rbf_need) + 1) & ~1;
    c->step_smem = ((size_t)state_d * P.G + (size_t)P.G * (8 * P.nK + 2 * P.eb_size + c->step_scr)) * 8;
    c->kkt_fb_stride = (size_t)((P.nK * (P.nK + 1) + 6 * P.nK + 31) & ~31);
    if (kern->dd_step2 && raise_smem_limit(kern->dd_step2, c->step_smem) != cudaSuccess)
      return bail(fail(DDNM_ECUDA, "cannot reserve dynamic shared memory"));
  }
  if (raise_smem_limit(kern->solve, c->smem) != cudaSuccess ||
      raise_smem_limit(kern->eval, c->smem) != cudaSuccess ||
      raise_smem_limit(kern->dd_eval, c->smem) != cudaSuccess ||
      raise_smem_limit(kern->dd_step, c->smem) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "cannot reserve dynamic shared memory"));
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern->solve, c->threads, c->smem) != cudaSuccess || occ < 1)
    return bail(fail(DDNM_ECUDA, "kernel does not fit on an SM"));
  c->ctas = occ * c->sms;
  if (cudaMalloc(&c->work, 4 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->counters, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "cudaMalloc failed"));
  // batch-wide evaluation program (lane = mu), when the instance is eligible
  std::vector<ddnm::WideHostRows> whr(a->n_blocks);
  for (int b = 0; b < a->n_blocks; ++b)
    whr[b] = ddnm::WideHostRows{hrows[b].src.data(), hrows[b].sgu.data(), hrows[b].sgv.data(),
                                hrows[b].nent.data(), hrows[b].bxc.data(), hrows[b].byc.data(),
                                hrows[b].cdc.data()};
  if (ddnm::wide_build(a, P, whr.data(), c->sms, &c->wide, c->wide_why) != 0)
    return bail(fail(DDNM_ECUDA, "cannot upload the wide evaluation tables"));
  *out = c;
  return 0;
}

int ddnm_plan_units(const ddnm_artifacts* a, int32_t* n_units, int32_t* row_unit,
                    int32_t* unit_info) {
  if (!a || !n_units) return fail(DDNM_EINVAL, "null argument");
  if (a->abi_version != DDNM_ABI_VERSION) return fail(DDNM_EINVAL, "ABI version mismatch");
  if (a->n_blocks < 1 || a->n_blocks > MAXB) return fail(DDNM_EINVAL, "need 1..16 blocks");
  *n_units = 0;
  if (!wants_units(a)) return 0;
  const UnitLimits L = unit_limits();
  int rc, u = 0, row_off = 0;
  for (int b = 0; b < a->n_blocks; ++b) {
    const ddnm_block& k = a->blocks[b];
    HostRows hr;
    if ((rc = build_stencil(a, k, hr))) return rc;
    std::vector<HostUnit> hu;
    if ((rc = split_block(a, k, hr, L, hu))) return rc;
    for (const HostUnit& x : hu) {
      if (unit_info) {
        int32_t* r = unit_info + (size_t)u * 8;
        r[0] = b; r[1] = x.flags; r[2] = (int32_t)x.rows.size(); r[3] = x.in.d.n_out;
        r[4] = x.in.d.n_hidden; r[5] = x.ga.d.n_out; r[6] = x.ga.d.n_hidden;
        r[7] = x.CA.empty() ? 0 : (int32_t)(x.CA.size() / a->n_c);
      }
      if (row_unit)
        for (int m : x.row_map) row_unit[row_off + m] = u;
      ++u;
    }
    row_off += k.n_rows;
  }
  *n_units = u;
  return 0;
}

int ddnm_ctx_destroy(ddnm_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& kv : c->io) cudaFree(kv.second.first);
  if (c->gbv) cudaFree(c->gbv);
  if (c->gJ) cudaFree(c->gJ);
  if (c->gJg) cudaFree(c->gJg);
  if (c->kkt_g) cudaFree(c->kkt_g);
  if (c->eb_g) cudaFree(c->eb_g);
  if (c->work) cudaFree(c->work);
  if (c->counters) cudaFree(c->counters);
  if (c->prof) cudaFree(c->prof);
  if (c->d_jobs) cudaFree(c->d_jobs);
  for (DdBuffers& b : c->dd_pool) b.release();
  if (c->wide) ddnm::wide_free(c->wide);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

int ddnm_ctx_info(const ddnm_ctx* c, ddnm_info* i) {
  if (!c || !i) return fail(DDNM_EINVAL, "null argument");
  i->n_primal = c->n_D;
  i->n_mult = c->n_C;
  i->n_blocks = c->nb;
  i->total_rows = c->tot_rows;
  i->total_out_rows = c->P.tot_out;
  i->total_out_R = c->P.tot_outR;
  i->total_int_out = c->tot_iout;
  i->total_gam_out = c->tot_gout;
  i->total_R = c->tot_R;
  i->total_cjac = c->tot_cjac;
  i->total_int_J = c->tot_intJ;
  i->total_gam_J = c->tot_gamJ;
  i->slots_per_cta = c->P.G;
  i->ctas = c->ctas;
  i->smem_bytes = (int32_t)c->smem;
  i->device = c->device;
  i->eval_units = c->n_units;
  i->wide = c->wide ? 1 : 0;
  return 0;
}

static int ensure_gbv(ddnm_ctx* c, size_t slots) {
  if (c->gbv_slots >= slots) return 0;
  // growing: work queued earlier (device entry points are asynchronous on
  // the caller's stream) may still use the old buffers
  if (c->gbv_slots) CUDA_TRY(cudaDeviceSynchronize());
  if (c->gbv) cudaFree(c->gbv);
  if (c->gJ) cudaFree(c->gJ);
  c->gbv = nullptr;
  c->gJ = nullptr;
  slots = std::max<size_t>(slots, 1);
  CUDA_TRY(cudaMalloc(&c->gbv, slots * c->tot_rows * 3 * sizeof(double)));
  CUDA_TRY(cudaMalloc(&c->gJ, slots * std::max(c->P.gJ_stride, 1) * sizeof(double)));
  if (c->gJg) cudaFree(c->gJg);
  c->gJg = nullptr;
  CUDA_TRY(cudaMalloc(&c->gJg, slots * std::max(c->P.gJg_stride, 1) * sizeof(double)));
  if (c->kkt_g) cudaFree(c->kkt_g);
  c->kkt_g = nullptr;
  if (c->kkt_stride) CUDA_TRY(cudaMalloc(&c->kkt_g, slots * c->kkt_stride * sizeof(double)));
  if (c->eb_g) cudaFree(c->eb_g);
  c->eb_g = nullptr;
  if (c->ebg) CUDA_TRY(cudaMalloc(&c->eb_g, slots * 2 * (size_t)c->P.eb_size * sizeof(double)));
  c->gbv_slots = slots;
  return 0;
}

static int fill_nan(cudaStream_t s, double* p, size_t n) {
  if (!p || n == 0) return 0;
  k_fill<<<148, 256, 0, s>>>(p, n, NAN);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

static int solve_wide(ddnm_ctx* c, int32_t B, const double* d_mu, const double* d_x0,
                      const double* d_lam0, const ddnm_sqp_cfg* cfg, ddnm_solve_out* o,
                      cudaStream_t s);

// which engine solves a batch: the persistent kernel (one slot per mu) or the
// round-synchronous batch-wide kernels (one lane per mu, ddnm_wide.h).
// DDNM_WIDE=0/1 forces; otherwise wide from DDNM_WIDE_MIN_B mu on (default:
// see wide_min_batch) when the instance is eligible.
static int wide_min_batch() {
  if (const char* e = getenv("DDNM_WIDE_MIN_B")) return atoi(e);
  return 1;
}
static bool use_wide(const ddnm_ctx* c, int B) {
  if (!c->wide || c->engine == DDNM_ENGINE_SLOTS) return false;
  if (B >= (1 << 23)) return false;     // lane entries hold mu in 24 bits (candidate index above)
  if (c->engine == DDNM_ENGINE_WIDE) return true;
  if (const char* e = getenv("DDNM_WIDE")) return atoi(e) != 0;
  return B >= wide_min_batch();
}

int ddnm_solve_batch_device(ddnm_ctx* c, int32_t B, const double* d_mu, const double* d_x0,
                            const double* d_lam0, const ddnm_sqp_cfg* cfg, ddnm_solve_out* o,
                            void* stream) {
  if (!c || !cfg || !o || !d_mu || !o->x || !o->lam) return fail(DDNM_EINVAL, "null argument");
  if (B < 0) return fail(DDNM_EINVAL, "negative batch");
  if (c->engine == DDNM_ENGINE_WIDE && !c->wide)
    return fail(DDNM_EUNSUPPORTED, "instance not eligible for the wide engine: " + c->wide_why);
  if (B > 0 && use_wide(c, B)) {
    CUDA_TRY(cudaSetDevice(c->device));
    const int rc = solve_wide(c, B, d_mu, d_x0, d_lam0, cfg, o, stream ? (cudaStream_t)stream : c->stream);
    // the wide engine's scratch grows with the batch (g / J lines of every
    // lane): when it does not fit, AUTO solves with the persistent kernel
    if (rc != DDNM_ENOMEM || c->engine == DDNM_ENGINE_WIDE) return rc;
    cudaGetLastError();
  }
  if (!(cfg->tol > 0) || cfg->max_iter < 1 || !(cfg->armijo_c1 > 0) || !(cfg->backtrack_factor > 0) ||
      !(cfg->backtrack_factor < 1) || cfg->max_halvings < 0)
    return fail(DDNM_EINVAL, "invalid solver configuration");
  if (!d_x0 && c->P.rbf_P == 0) return fail(DDNM_EINVAL, "instance has no fitted initializer");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (B == 0) return 0;
  const int ctas = std::min(c->ctas, (B + c->P.G - 1) / c->P.G);
  int rc;
  if ((rc = ensure_gbv(c, (size_t)ctas * c->P.G))) return rc;
  Params P = c->P;
  P.B = B;
  P.mu = d_mu;
  P.x0_in = d_x0;
  P.lam0_in = d_lam0;
  P.cfg.tol = cfg->tol;
  P.cfg.c1 = cfg->armijo_c1;
  P.cfg.factor = cfg->backtrack_factor;
  P.cfg.reg_scale = cfg->reg_scale;
  P.cfg.max_iter = cfg->max_iter;
  P.cfg.max_halvings = cfg->max_halvings;
  P.so.x = o->x; P.so.lam = o->lam; P.so.merit = o->merit; P.so.objective = o->objective;
  P.so.merit_hist = o->merit_hist; P.so.obj_hist = o->obj_hist; P.so.alpha_hist = o->alpha_hist;
  P.so.x0 = o->x0; P.so.lam0 = o->lam0;
  P.so.n_iter = o->n_iter; P.so.n_evals = o->n_evals; P.so.status = o->status; P.so.n_reg = o->n_reg;
  P.gbv = c->gbv;
  P.gJ = c->gJ;
  P.gJg = c->gJg;
  P.kkt_g = c->kkt_g;
  P.eb_glob = c->eb_g;
  P.work = c->work;
  P.counters = c->counters;
  P.prof = nullptr;
  if (getenv("DDNM_PROF")) {
    if (!c->prof) CUDA_TRY(cudaMalloc(&c->prof, 16 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(c->prof, 0, 16 * sizeof(unsigned long long), s));
    P.prof = c->prof;
  }
  if ((rc = fill_nan(s, o->merit_hist, (size_t)B * (cfg->max_iter + 1)))) return rc;
  if ((rc = fill_nan(s, o->obj_hist, (size_t)B * (cfg->max_iter + 1)))) return rc;
  if ((rc = fill_nan(s, o->alpha_hist, (size_t)B * cfg->max_iter))) return rc;
  CUDA_TRY(cudaMemsetAsync(c->work, 0, 4 * sizeof(int), s));
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(unsigned long long), s));
  void* args[] = {&P};
  CUDA_TRY(cudaLaunchKernel(c->K.solve, dim3(ctas), dim3(c->threads), args, c->smem, s));
  c->last_rounds = 0;
  c->last_launches = 1;
  c->last_lanes = 0;
  return 0;
}

int ddnm_ctx_set_engine(ddnm_ctx* c, int32_t engine) {
  if (!c) return fail(DDNM_EINVAL, "null argument");
  if (engine < DDNM_ENGINE_AUTO || engine > DDNM_ENGINE_WIDE) return fail(DDNM_EINVAL, "unknown engine");
  if (engine == DDNM_ENGINE_WIDE && !c->wide)
    return fail(DDNM_EUNSUPPORTED, "instance not eligible for the wide engine: " + c->wide_why);
  c->engine = engine;
  return 0;
}

int ddnm_last_rounds(const ddnm_ctx* c, int64_t* rounds, int64_t* launches) {
  if (!c) return fail(DDNM_EINVAL, "null argument");
  if (rounds) *rounds = c->last_rounds;
  if (launches) *launches = c->last_launches;
  return 0;
}

int ddnm_last_lanes(const ddnm_ctx* c, int64_t* lanes) {
  if (!c || !lanes) return fail(DDNM_EINVAL, "null argument");
  *lanes = c->last_lanes;
  return 0;
}

extern "C" int ddnm_last_profile(const ddnm_ctx* c, uint64_t* cycles16) {
  if (!c || !cycles16) return fail(DDNM_EINVAL, "null argument");
  if (!c->prof) { for (int i = 0; i < 16; ++i) cycles16[i] = 0; return 0; }
  CUDA_TRY(cudaMemcpy(cycles16, c->prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return 0;
}

int ddnm_last_counters(const ddnm_ctx* c, int64_t* evals, int64_t* kkts) {
  if (!c) return fail(DDNM_EINVAL, "null argument");
  unsigned long long h[2] = {0, 0};
  CUDA_TRY(cudaMemcpy(h, c->counters, sizeof h, cudaMemcpyDeviceToHost));
  if (evals) *evals = (int64_t)h[0];
  if (kkts) *kkts = (int64_t)h[1];
  return 0;
}

int ddnm_solve_batch(ddnm_ctx* c, int32_t B, const double* mu, const double* x0, const double* lam0,
                     const ddnm_sqp_cfg* cfg, ddnm_solve_out* o) {
  if (!c || !cfg || !o || !mu || !o->x || !o->lam) return fail(DDNM_EINVAL, "null argument");
  if (B <= 0) return B == 0 ? 0 : fail(DDNM_EINVAL, "negative batch");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t nD = c->n_D, nC = c->n_C, K1 = cfg->max_iter + 1, K = cfg->max_iter;
  cudaStream_t s = c->stream;
  struct Field { const char* name; void* host; size_t bytes; bool in; };
  ddnm_solve_out d{};
  void* dmu = nullptr; void* dx0 = nullptr; void* dl0 = nullptr;
  int rc;
  if ((rc = io_buf(c, "mu", B * 2 * 8, &dmu))) return rc;
  CUDA_TRY(cudaMemcpyAsync(dmu, mu, B * 2 * 8, cudaMemcpyHostToDevice, s));
  if (x0) {
    if ((rc = io_buf(c, "x0in", B * nD * 8, &dx0))) return rc;
    CUDA_TRY(cudaMemcpyAsync(dx0, x0, B * nD * 8, cudaMemcpyHostToDevice, s));
  }
  if (lam0) {
    if ((rc = io_buf(c, "l0in", B * nC * 8, &dl0))) return rc;
    CUDA_TRY(cudaMemcpyAsync(dl0, lam0, B * nC * 8, cudaMemcpyHostToDevice, s));
  }
  Field f[] = {
      {"x", o->x, B * nD * 8, false},           {"lam", o->lam, B * nC * 8, false},
      {"n_iter", o->n_iter, B * 4ul, false},    {"n_evals", o->n_evals, B * 4ul, false},
      {"status", o->status, B * 4ul, false},    {"n_reg", o->n_reg, B * 4ul, false},
      {"merit", o->merit, B * 8ul, false},      {"objective", o->objective, B * 8ul, false},
      {"merit_hist", o->merit_hist, B * K1 * 8, false}, {"obj_hist", o->obj_hist, B * K1 * 8, false},
      {"alpha_hist", o->alpha_hist, B * K * 8, false},  {"x0", o->x0, B * nD * 8, false},
      {"lam0", o->lam0, B * nC * 8, false},
  };
  void* dp[13];
  for (int i = 0; i < 13; ++i) {
    dp[i] = nullptr;
    if (f[i].host && (rc = io_buf(c, std::string("o_") + f[i].name, f[i].bytes, &dp[i]))) return rc;
  }
  d.x = (double*)dp[0]; d.lam = (double*)dp[1]; d.n_iter = (int*)dp[2]; d.n_evals = (int*)dp[3];
  d.status = (int*)dp[4]; d.n_reg = (int*)dp[5]; d.merit = (double*)dp[6]; d.objective = (double*)dp[7];
  d.merit_hist = (double*)dp[8]; d.obj_hist = (double*)dp[9]; d.alpha_hist = (double*)dp[10];
  d.x0 = (double*)dp[11]; d.lam0 = (double*)dp[12];
  if ((rc = ddnm_solve_batch_device(c, B, (double*)dmu, (double*)dx0, (double*)dl0, cfg, &d, s))) return rc;
  for (int i = 0; i < 13; ++i)
    if (f[i].host) CUDA_TRY(cudaMemcpyAsync(f[i].host, dp[i], f[i].bytes, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int ddnm_eval_batch(ddnm_ctx* c, int32_t B, const double* mu, const double* x, const double* lam,
                    double reg_scale, ddnm_eval_out* o) {
  if (!c || !o || !mu || !x || !lam) return fail(DDNM_EINVAL, "null argument");
  if (B <= 0) return B == 0 ? 0 : fail(DDNM_EINVAL, "negative batch");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const size_t nD = c->n_D, nC = c->n_C;
  int rc;
  void *dmu, *dx, *dl;
  if ((rc = io_buf(c, "mu", B * 2 * 8, &dmu)) || (rc = io_buf(c, "ex", B * nD * 8, &dx)) ||
      (rc = io_buf(c, "el", B * nC * 8, &dl)))
    return rc;
  CUDA_TRY(cudaMemcpyAsync(dmu, mu, B * 2 * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dx, x, B * nD * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dl, lam, B * nC * 8, cudaMemcpyHostToDevice, s));
  struct Field { const char* name; void* host; size_t bytes; };
  Field f[] = {
      {"rho", o->rho, B * nD * 8},
      {"con", o->con, B * nC * 8},
      {"merit", o->merit, B * 8ul},
      {"objective", o->objective, B * 8ul},
      {"Br", o->Br, B * (size_t)c->P.tot_out * 8},
      {"R", o->R, B * (size_t)c->P.tot_outR * 8},
      {"cval", o->cval, B * (size_t)c->nb * nC * 8},
      {"cjac", o->cjac, B * (size_t)c->tot_cjac * 8},
      {"int_g", o->int_g, B * (size_t)c->tot_iout * 8},
      {"int_J", o->int_J, B * (size_t)c->tot_intJ * 8},
      {"gam_g", o->gam_g, B * (size_t)c->tot_gout * 8},
      {"gam_J", o->gam_J, B * (size_t)c->tot_gamJ * 8},
      {"bvals", o->bvals, B * (size_t)c->tot_rows * 3 * 8},
      {"step", o->step, B * (nD + nC) * 8},
      {"kkt_status", o->kkt_status, B * 4ul},
  };
  constexpr int NF = 15;
  void* dp[NF];
  for (int i = 0; i < NF; ++i) {
    dp[i] = nullptr;
    if (f[i].host && (rc = io_buf(c, std::string("e_") + f[i].name, f[i].bytes, &dp[i]))) return rc;
  }
  const int G = c->P.G;
  const int ctas = (B + G - 1) / G;
  if ((rc = ensure_gbv(c, (size_t)ctas * G))) return rc;
  Params P = c->P;
  P.B = B;
  P.mu = (double*)dmu;
  P.x0_in = (double*)dx;
  P.lam0_in = (double*)dl;
  P.cfg.reg_scale = reg_scale;
  P.eo.rho = (double*)dp[0]; P.eo.con = (double*)dp[1]; P.eo.merit = (double*)dp[2];
  P.eo.objective = (double*)dp[3]; P.eo.Br = (double*)dp[4]; P.eo.R = (double*)dp[5];
  P.eo.cval = (double*)dp[6]; P.eo.cjac = (double*)dp[7]; P.eo.int_g = (double*)dp[8];
  P.eo.int_J = (double*)dp[9]; P.eo.gam_g = (double*)dp[10]; P.eo.gam_J = (double*)dp[11];
  P.eo.bvals = (double*)dp[12]; P.eo.step = (double*)dp[13]; P.eo.kkt_status = (int*)dp[14];
  P.eval_mode = 1;
  P.eval_step = (o->step || o->kkt_status) ? 1 : 0;
  P.gbv = c->gbv;
  P.gJ = c->gJ;
  P.gJg = c->gJg;
  P.kkt_g = c->kkt_g;
  P.eb_glob = c->eb_g;
  P.work = c->work;
  P.counters = c->counters;
  void* args[] = {&P};
  CUDA_TRY(cudaLaunchKernel(c->K.eval, dim3(ctas), dim3(c->threads), args, c->smem, s));
  for (int i = 0; i < NF; ++i)
    if (f[i].host) CUDA_TRY(cudaMemcpyAsync(f[i].host, dp[i], f[i].bytes, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int ddnm_ctx_set_full_decoders(ddnm_ctx* c, const ddnm_decoder* interior,
                               const ddnm_decoder* interface) {
  if (!c || !interior) return fail(DDNM_EINVAL, "null argument");
  if (c->P.con_mode == DDNM_CON_SRPC && !interface)
    return fail(DDNM_EINVAL, "SRPC needs the full interface maps");
  CUDA_TRY(cudaSetDevice(c->device));
  int rc;
  const int nb = c->nb;
  for (int b = 0; b < nb; ++b) {
    if ((rc = check_decoder(interior[b], c->P.blk[b].ni, c->map_kind, "full interior"))) return rc;
    if (interface && (rc = check_decoder(interface[b], c->P.blk[b].ng, c->map_kind, "full interface")))
      return rc;
  }
  std::vector<DecodeJob> jobs(2 * nb);
  int off = 0, max_h = 0;
  for (int b = 0; b < nb; ++b) {
    const BlockDev& B = c->P.blk[b];
    HostWindows hw;
    DecodeJob& ji = jobs[2 * b];
    if ((rc = upload_decoder(c, interior[b], B.ni, c->map_kind, B.in.act, ji.D, hw))) return rc;
    ji.x_off = B.xoff; ji.lat = B.ni; ji.out_off = off;
    off += ji.D.n_out;
    DecodeJob& jg = jobs[2 * b + 1];
    if (interface) {
      if ((rc = upload_decoder(c, interface[b], B.ng, c->map_kind, B.ga.act, jg.D, hw))) return rc;
    } else {
      jg.D = B.ga;
    }
    jg.x_off = B.xoff + B.ni; jg.lat = B.ng; jg.out_off = off;
    off += jg.D.n_out;
    max_h = std::max({max_h, ji.D.n_hidden, jg.D.n_hidden});
  }
  const int mu = c->map_kind == DDNM_MAP_LINEAR ? 8 : decode_mu_tile(max_h, 200 * 1024);
  if (mu == 0) return fail(DDNM_EUNSUPPORTED, "decoder hidden layer too wide for shared memory");
  if (c->d_jobs) cudaFree(c->d_jobs);
  c->d_jobs = nullptr;
  CUDA_TRY(cudaMalloc(&c->d_jobs, jobs.size() * sizeof(DecodeJob)));
  CUDA_TRY(cudaMemcpy(c->d_jobs, jobs.data(), jobs.size() * sizeof(DecodeJob), cudaMemcpyHostToDevice));
  c->state_len = off;
  c->dec_max_hidden = max_h;
  c->dec_mu_tile = mu;
  return 0;
}

int ddnm_ctx_state_len(const ddnm_ctx* c, int64_t* len) {
  if (!c || !len) return fail(DDNM_EINVAL, "null argument");
  *len = c->state_len;
  return 0;
}

int ddnm_decode_batch_device(ddnm_ctx* c, int32_t B, const double* d_x, const double* d_fom,
                             double* d_states, double* d_err, void* stream) {
  if (!c || !d_x) return fail(DDNM_EINVAL, "null argument");
  if (B < 0) return fail(DDNM_EINVAL, "negative batch");
  if (!c->d_jobs) return fail(DDNM_EINVAL, "no full decoders (ddnm_ctx_set_full_decoders)");
  if ((d_fom == nullptr) != (d_err == nullptr)) return fail(DDNM_EINVAL, "fom and err go together");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (B == 0) return 0;
  DecodeParams p{};
  p.jobs = c->d_jobs;
  p.n_jobs = 2 * c->nb;
  p.nb = c->nb;
  p.B = B;
  p.n_D = c->n_D;
  p.state_len = c->state_len;
  p.act = c->P.act;
  p.linear = c->map_kind == DDNM_MAP_LINEAR;
  p.mu_tile = c->dec_mu_tile;
  p.max_hidden = c->dec_max_hidden;
  p.x = d_x;
  p.fom = d_fom;
  p.states = d_states;
  p.err = d_err;
  int rc;
  if (d_fom) {
    void* part = nullptr;
    if ((rc = io_buf(c, "dec_part", (size_t)B * p.n_jobs * 2 * 8, &part))) return rc;
    p.part = (double*)part;
  }
  CUDA_TRY(launch_decode(p, s));
  return 0;
}

int ddnm_decode_batch(ddnm_ctx* c, int32_t B, const double* x, const double* fom, double* states,
                      double* err) {
  if (!c || !x) return fail(DDNM_EINVAL, "null argument");
  if (B <= 0) return B == 0 ? 0 : fail(DDNM_EINVAL, "negative batch");
  if (!c->d_jobs) return fail(DDNM_EINVAL, "no full decoders (ddnm_ctx_set_full_decoders)");
  if ((fom == nullptr) != (err == nullptr)) return fail(DDNM_EINVAL, "fom and err go together");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const size_t L = (size_t)c->state_len * B * 8;
  void *dx, *df = nullptr, *ds = nullptr, *de = nullptr;
  int rc;
  if ((rc = io_buf(c, "dec_x", (size_t)B * c->n_D * 8, &dx))) return rc;
  CUDA_TRY(cudaMemcpyAsync(dx, x, (size_t)B * c->n_D * 8, cudaMemcpyHostToDevice, s));
  if (fom) {
    if ((rc = io_buf(c, "dec_fom", L, &df)) || (rc = io_buf(c, "dec_err", (size_t)B * 8, &de))) return rc;
    CUDA_TRY(cudaMemcpyAsync(df, fom, L, cudaMemcpyHostToDevice, s));
  }
  if (states && (rc = io_buf(c, "dec_states", L, &ds))) return rc;
  if ((rc = ddnm_decode_batch_device(c, B, (double*)dx, (double*)df, (double*)ds, (double*)de, s)))
    return rc;
  if (states) CUDA_TRY(cudaMemcpyAsync(states, ds, L, cudaMemcpyDeviceToHost, s));
  if (err) CUDA_TRY(cudaMemcpyAsync(err, de, (size_t)B * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return 0;
}


// ---- subdomain-sharded round-synchronous solve ----------

}  // extern "C"

struct ddnm_dd {
  ddnm_ctx* c = nullptr;
  Params P{};
  int B = 0, ctas = 0;
  // per-solve state and copies of the context's per-slot scratch (boundary
  // values, Jacobian rows, KKT workspace, evaluation buffers when in L2,
  // own trial records): a sharded solve never shares them with another
  // solve on the same context; taken from / returned to the context's pool
  DdBuffers buf;
  cudaStream_t stream = nullptr;  // the caller's stream of the last call
  bool wide = false;              // evaluations by the batch-wide kernels (ddnm_wide.h)
  bool wide_by_mu = false;        // ... one candidate per mu, packets by mu (sharded ranks)
  size_t wide_pk_cap = 0;         // doubles in the caller's packet buffer when known
  const void* step_kern = nullptr; // step kernel / shared memory of the wide solve (null: the context's)
  size_t step_smem = 0;
};

namespace {
int eb_span(const ddnm_ctx* c, int lo, int hi, int* off) {
  const Params& P = c->P;
  if (lo < 0 || hi > P.nb || lo >= hi) return fail(DDNM_EINVAL, "empty or out-of-range block range");
  *off = P.blk[lo].eb_off;
  return (hi < P.nb ? P.blk[hi].eb_off : P.eb_rho) - *off;
}

int dd_run(ddnm_dd* d, const void* kern, cudaStream_t s, int32_t* n_active, int ctas = 0) {
  ddnm_ctx* c = d->c;
  CUDA_TRY(cudaMemsetAsync(d->buf.active, 0, sizeof(int), s));
  void* args[] = {&d->P};
  if (ctas == 0) ctas = d->ctas;
  size_t smem = c->smem;
  if (kern == c->K.dd_step && d->step_kern && !d->P.dd_init) { kern = d->step_kern; smem = d->step_smem; }
  if (ctas > 0)
    CUDA_TRY(cudaLaunchKernel(kern, dim3(ctas), dim3(c->threads), args, smem, s));
  if (getenv("DDNM_WIDE_SYNC")) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
      fprintf(stderr, "ddnm: %s (init %d, %d CTAs, B %d) failed: %s\n",
              kern == c->K.dd_step ? "k_dd_step" : "k_dd_eval", d->P.dd_init, ctas, d->P.B,
              cudaGetErrorString(e));
  }
  if (n_active) {
    int h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, d->buf.active, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *n_active = h;
  }
  return 0;
}
}  // namespace

extern "C" {

int ddnm_dd_packet_len(const ddnm_ctx* c, int32_t blk_lo, int32_t blk_hi, int64_t* len) {
  if (!c || !len) return fail(DDNM_EINVAL, "null argument");
  int off = 0;
  const int n = eb_span(c, blk_lo, blk_hi, &off);
  if (n < 0) return n;
  *len = n;
  return 0;
}

int ddnm_dd_begin(ddnm_ctx* c, int32_t B, const double* d_mu, const double* d_x0,
                  const double* d_lam0, const ddnm_sqp_cfg* cfg, int32_t blk_lo, int32_t blk_hi,
                  const ddnm_solve_out* o, void* stream, ddnm_dd** out, int32_t* n_active) {
  if (!c || !cfg || !o || !out || !d_mu || !o->x || !o->lam) return fail(DDNM_EINVAL, "null argument");
  *out = nullptr;
  if (B < 1) return fail(DDNM_EINVAL, "batch must be positive");
  if (!(cfg->tol > 0) || cfg->max_iter < 1 || !(cfg->armijo_c1 > 0) || !(cfg->backtrack_factor > 0) ||
      !(cfg->backtrack_factor < 1) || cfg->max_halvings < 0)
    return fail(DDNM_EINVAL, "invalid solver configuration");
  if (!d_x0 && c->P.rbf_P == 0) return fail(DDNM_EINVAL, "instance has no fitted initializer");
  int off = 0;
  int rc = eb_span(c, blk_lo, blk_hi, &off);
  if (rc < 0) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  auto* d = new ddnm_dd();
  d->stream = s;
  d->c = c;
  d->B = B;
  d->ctas = (B + c->P.G - 1) / c->P.G;
  auto bail = [&](int r) { ddnm_dd_end(d); return r; };
  const int rec = (c->P.n_D + 1 + 1) & ~1;
  // buffers: the smallest pooled set that holds B mu, else new ones
  {
    int best = -1;
    for (int i = 0; i < (int)c->dd_pool.size(); ++i)
      if (c->dd_pool[i].cap >= B && (best < 0 || c->dd_pool[i].cap < c->dd_pool[best].cap)) best = i;
    if (best >= 0) {
      d->buf = c->dd_pool[best];
      c->dd_pool.erase(c->dd_pool.begin() + best);
    }
  }
  DdBuffers& bf = d->buf;
  if (bf.cap < B) {
    bf.release();
    bf.cap = B;
    // per-mu scratch (slot = mu); one CTA of spare slots for a step slice that
    // starts mid-CTA (k_dd_step maps mu_lo + blockIdx.x * G + s)
    const size_t slots = (size_t)(d->ctas + 1) * c->P.G;
    if (cudaMalloc(&bf.gbv, slots * std::max(c->tot_rows * 3, 1) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&bf.gJ, slots * std::max(c->P.gJ_stride, 1) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&bf.gJg, slots * std::max(c->P.gJg_stride, 1) * sizeof(double)) != cudaSuccess ||
        (c->kkt_stride && cudaMalloc(&bf.kkt_g, slots * c->kkt_stride * sizeof(double)) != cudaSuccess) ||
        (c->ebg && cudaMalloc(&bf.eb_g, slots * 2 * (size_t)c->P.eb_size * sizeof(double)) != cudaSuccess))
      return bf.release(), bail(fail(DDNM_ENOMEM, "cannot allocate the sharded solve scratch"));
    if (cudaMalloc(&bf.st, (size_t)B * sizeof(SlotState)) != cudaSuccess ||
        cudaMalloc(&bf.vec, (size_t)B * 8 * c->P.nK * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&bf.ecur, (size_t)B * c->P.eb_size * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&bf.active, sizeof(int)) != cudaSuccess)
      return bf.release(), bail(fail(DDNM_ENOMEM, "cannot allocate the sharded solve state"));
    if (cudaMalloc(&bf.trials, (size_t)B * rec * sizeof(double)) != cudaSuccess)
      return bf.release(), bail(fail(DDNM_ENOMEM, "cannot allocate the trial records"));
  }
  Params& P = d->P;
  P = c->P;
  P.B = B;
  P.mu = d_mu;
  P.x0_in = d_x0;
  P.lam0_in = d_lam0;
  P.cfg.tol = cfg->tol;
  P.cfg.c1 = cfg->armijo_c1;
  P.cfg.factor = cfg->backtrack_factor;
  P.cfg.reg_scale = cfg->reg_scale;
  P.cfg.max_iter = cfg->max_iter;
  P.cfg.max_halvings = cfg->max_halvings;
  P.so.x = o->x; P.so.lam = o->lam; P.so.merit = o->merit; P.so.objective = o->objective;
  P.so.merit_hist = o->merit_hist; P.so.obj_hist = o->obj_hist; P.so.alpha_hist = o->alpha_hist;
  P.so.x0 = o->x0; P.so.lam0 = o->lam0;
  P.so.n_iter = o->n_iter; P.so.n_evals = o->n_evals; P.so.status = o->status; P.so.n_reg = o->n_reg;
  P.gbv = bf.gbv;
  P.gJ = bf.gJ;
  P.gJg = bf.gJg;
  P.kkt_g = bf.kkt_g;
  P.eb_glob = bf.eb_g;
  P.work = c->work;
  P.counters = c->counters;
  P.prof = nullptr;
  if (getenv("DDNM_PROF")) {           // phase clocks of the step kernel
    if (!c->prof && cudaMalloc(&c->prof, 16 * sizeof(unsigned long long)) != cudaSuccess)
      return bail(fail(DDNM_ECUDA, "cudaMalloc failed"));
    if (cudaMemsetAsync(c->prof, 0, 16 * sizeof(unsigned long long), s) != cudaSuccess)
      return bail(fail(DDNM_ECUDA, "memset failed"));
    P.prof = c->prof;
  }
  P.b_lo = blk_lo;
  P.b_hi = blk_hi;
  P.dd_st = bf.st;
  P.dd_vec = bf.vec;
  P.dd_ecur = bf.ecur;
  P.dd_active = bf.active;
  P.dd_trial = bf.trials;
  P.dd_rec = rec;
  P.dd_mu_lo = 0;
  P.dd_mu_hi = B;
  if ((rc = fill_nan(s, o->merit_hist, (size_t)B * (cfg->max_iter + 1)))) return bail(rc);
  if ((rc = fill_nan(s, o->obj_hist, (size_t)B * (cfg->max_iter + 1)))) return bail(rc);
  if ((rc = fill_nan(s, o->alpha_hist, (size_t)B * cfg->max_iter))) return bail(rc);
  if (cudaMemsetAsync(c->counters, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "memset failed"));
  P.dd_init = 1;
  if ((rc = dd_run(d, c->K.dd_step, s, n_active))) return bail(rc);
  P.dd_init = 0;
  *out = d;
  return 0;
}

int ddnm_dd_eval(ddnm_dd* d, double* d_packets, int64_t pk_stride, void* stream) {
  if (!d || !d_packets) return fail(DDNM_EINVAL, "null argument");
  int off = 0;
  const int len = eb_span(d->c, d->P.b_lo, d->P.b_hi, &off);
  if (pk_stride < len) return fail(DDNM_EINVAL, "packet stride shorter than this rank's packet");
  CUDA_TRY(cudaSetDevice(d->c->device));
  cudaStream_t s = (cudaStream_t)stream;
  d->stream = s;
  d->P.dd_pk = d_packets;
  d->P.pk_stride = (int)pk_stride;
  if (d->wide) {
    if (!d->wide_by_mu && (size_t)pk_stride * ddnm::wide_packet_rows(d->buf.wide) > d->wide_pk_cap &&
        d->wide_pk_cap)
      return fail(DDNM_EINVAL, "packet buffer smaller than one row per lane");
    if (ddnm::wide_eval(d->c->wide, d->P, d->buf.wide, d_packets, (int)pk_stride, d->wide_by_mu, s) != 0)
      return fail(DDNM_ECUDA, "wide evaluation launch failed");
    return 0;
  }
  return dd_run(d, d->c->K.dd_eval, s, nullptr);
}

/* Switch a sharded solve that owns every block to the batch-wide evaluation
 * kernels (ddnm_wide.h): same packets to rounding, one lane per mu. */
int ddnm_dd_set_wide(ddnm_dd* d, int32_t on) {
  if (!d) return fail(DDNM_EINVAL, "null argument");
  if (!on) {
    d->wide = false; d->P.dd_vbase = nullptr; d->P.dd_kof = nullptr;
    d->P.scr_size = d->c->P.scr_size; d->P.kkt_fb = nullptr; d->step_kern = nullptr;
    return 0;
  }
  ddnm_ctx* c = d->c;
  if (!c->wide) return fail(DDNM_EUNSUPPORTED, "instance not eligible for the wide evaluation: " + c->wide_why);
  const bool by_mu = on == 2;
  if (!by_mu && (d->P.b_lo != 0 || d->P.b_hi != d->P.nb))
    return fail(DDNM_EUNSUPPORTED, "the wide evaluation with candidates needs every block on this rank "
                                   "(use mode 2: one packet per mu)");
  CUDA_TRY(cudaSetDevice(c->device));
  std::string err;
  if (ddnm::wide_alloc(c->wide, d->B, &d->buf.wide, err) != 0) return fail(DDNM_ENOMEM, err);
  if (ddnm::wide_begin(c->wide, d->P, d->buf.wide, d->stream) != 0)
    return fail(DDNM_ECUDA, "wide boundary-value launch failed");
  d->P.dd_vbase = by_mu ? nullptr : d->buf.wide.vbase;
  d->P.dd_kof = by_mu ? nullptr : d->buf.wide.kof;
  d->wide_by_mu = by_mu;
  // the step kernel runs alone: KKT-sized shared scratch, dense fallback in a
  // global workspace, two CTAs per SM when compiled (DDNM_STEP2=0: the plain one)
  if (c->step_scr > 0 && !getenv("DDNM_STEP_FULL")) {
    DdBuffers& bf = d->buf;
    if (!bf.kkt_fb &&
        cudaMalloc(&bf.kkt_fb, (size_t)(bf.cap + 2 * c->P.G) * c->kkt_fb_stride * sizeof(double)) != cudaSuccess)
      return fail(DDNM_ENOMEM, "cannot allocate the KKT fallback workspace");
    d->P.scr_size = c->step_scr;
    d->P.kkt_fb = bf.kkt_fb;
    d->P.kkt_fb_stride = (long long)c->kkt_fb_stride;
    const char* e2 = getenv("DDNM_STEP2");
    const bool two = c->K.dd_step2 && !(e2 && atoi(e2) == 0);
    d->step_kern = two ? c->K.dd_step2 : c->K.dd_step;
    d->step_smem = c->step_smem;
  }
  d->wide = true;
  return 0;
}

int ddnm_dd_eval_p2p(ddnm_dd* d, double* const* peers, int32_t nranks, int32_t rank,
                     int64_t pk_stride, void* stream) {
  if (!d || !peers) return fail(DDNM_EINVAL, "null argument");
  if (nranks < 1 || nranks > MAXB || rank < 0 || rank >= nranks)
    return fail(DDNM_EINVAL, "need 1..16 ranks and 0 <= rank < nranks");
  int off = 0;
  const int len = eb_span(d->c, d->P.b_lo, d->P.b_hi, &off);
  if (pk_stride < len) return fail(DDNM_EINVAL, "packet stride shorter than this rank's packet");
  for (int r = 0; r < nranks; ++r)
    if (!peers[r]) return fail(DDNM_EINVAL, "null peer buffer");
  CUDA_TRY(cudaSetDevice(d->c->device));
  cudaStream_t s = (cudaStream_t)stream;
  d->stream = s;
  d->P.pk_stride = (int)pk_stride;
  d->P.dd_npeers = nranks;
  d->P.dd_rank = rank;
  for (int r = 0; r < nranks; ++r) d->P.dd_peers[r] = peers[r];
  const int rc = dd_run(d, d->c->K.dd_eval, s, nullptr);   // parameters copied at launch
  d->P.dd_npeers = 0;
  return rc;
}

int ddnm_dev_alloc(int32_t device, int64_t bytes, void** out) {
  if (!out || bytes <= 0) return fail(DDNM_EINVAL, "bad allocation request");
  *out = nullptr;
  if (device >= 0) CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaMalloc(out, (size_t)bytes));
  CUDA_TRY(cudaMemset(*out, 0, (size_t)bytes));
  return 0;
}

int ddnm_dev_free(void* p) {
  if (p) CUDA_TRY(cudaFree(p));
  return 0;
}

int ddnm_ipc_get_handle(const void* dptr, unsigned char* handle) {
  if (!dptr || !handle) return fail(DDNM_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  return 0;
}

int ddnm_ipc_open_handle(const unsigned char* handle, void** dptr) {
  if (!handle || !dptr) return fail(DDNM_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int ddnm_ipc_close_handle(void* dptr) {
  if (!dptr) return fail(DDNM_EINVAL, "null argument");
  CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return 0;
}

int ddnm_dd_step(ddnm_dd* d, const double* d_gathered, int32_t nranks, const int32_t* bounds,
                 int64_t pk_stride, void* stream, int32_t* n_active) {
  if (!d || !d_gathered || !bounds) return fail(DDNM_EINVAL, "null argument");
  const int nb = d->P.nb;
  if (nranks < 1 || nranks > nb) return fail(DDNM_EINVAL, "need 1..n_blocks ranks");
  if (bounds[0] != 0 || bounds[nranks] != nb) return fail(DDNM_EINVAL, "rank bounds must cover every block");
  for (int r = 0; r < nranks; ++r) {
    int off = 0;
    const int len = eb_span(d->c, bounds[r], bounds[r + 1], &off);
    if (len < 0) return len;
    if (len > pk_stride) return fail(DDNM_EINVAL, "packet stride shorter than a rank's packet");
  }
  CUDA_TRY(cudaSetDevice(d->c->device));
  cudaStream_t s = (cudaStream_t)stream;
  d->stream = s;
  d->P.dd_gath = d_gathered;
  d->P.dd_nranks = nranks;
  d->P.pk_stride = (int)pk_stride;
  for (int r = 0; r <= nranks; ++r) d->P.dd_bnd[r] = bounds[r];
  const int G = d->c->P.G;
  const int n = d->P.dd_mu_hi - d->P.dd_mu_lo;
  const int rc = dd_run(d, d->c->K.dd_step, s, nullptr, n > 0 ? (n + G - 1) / G : -1);
  if (rc) return rc;
  if (n_active) {
    int h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, d->buf.active, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *n_active = h;
  }
  return 0;
}

int ddnm_dd_trial_len(const ddnm_dd* d, int64_t* len) {
  if (!d || !len) return fail(DDNM_EINVAL, "null argument");
  *len = d->P.dd_rec;
  return 0;
}

int ddnm_dd_set_trials(ddnm_dd* d, double* d_trials, int64_t cap, int32_t mu_lo, int32_t mu_hi,
                       void* stream) {
  if (!d || !d_trials) return fail(DDNM_EINVAL, "null argument");
  if (cap < d->B) return fail(DDNM_EINVAL, "trial buffer holds fewer records than the batch");
  if (mu_lo < 0 || mu_hi < mu_lo || mu_hi > d->B) return fail(DDNM_EINVAL, "bad mu slice");
  CUDA_TRY(cudaSetDevice(d->c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rec = (size_t)d->P.dd_rec;
  if (d_trials != d->P.dd_trial) {
    CUDA_TRY(cudaMemcpyAsync(d_trials, d->P.dd_trial, (size_t)d->B * rec * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    if (cap > d->B)
      CUDA_TRY(cudaMemsetAsync(d_trials + (size_t)d->B * rec, 0,
                               (size_t)(cap - d->B) * rec * sizeof(double), s));
  }
  d->P.dd_trial = d_trials;
  d->P.dd_mu_lo = mu_lo;
  d->P.dd_mu_hi = mu_hi;
  return 0;
}

int ddnm_dd_end(ddnm_dd* d) {
  if (!d) return 0;
  cudaSetDevice(d->c->device);
  cudaStreamSynchronize(d->stream);
  // back to the context's pool (the next sharded solve skips the mallocs)
  if (d->buf.cap > 0) {
    if (d->c->dd_pool.size() < 4) d->c->dd_pool.push_back(d->buf);
    else d->buf.release();
  }
  delete d;
  return 0;
}

}  // extern "C"

// The whole batched solve as rounds of the batch-wide evaluation and the SQP
// step kernel (k_dd_step: Armijo decision, KKT solve, trial point), looped
// here: rounds are launched back to back and the running count is read every
// few rounds (rounds after the last mu finished are empty launches).
static int solve_wide(ddnm_ctx* c, int32_t B, const double* d_mu, const double* d_x0,
                      const double* d_lam0, const ddnm_sqp_cfg* cfg, ddnm_solve_out* o,
                      cudaStream_t s) {
  ddnm_dd* d = nullptr;
  int rc = ddnm_dd_begin(c, B, d_mu, d_x0, d_lam0, cfg, 0, c->nb, o, s, &d, nullptr);
  if (rc) return rc;
  auto bail = [&](int r) { const std::string keep = g_err; ddnm_dd_end(d); g_err = keep; return r; };
  if ((rc = ddnm_dd_set_wide(d, 1))) return bail(rc);
  int off = 0;
  const int stride = eb_span(c, 0, c->nb, &off);
  DdBuffers& bf = d->buf;
  const size_t pk_need = ddnm::wide_packet_rows(bf.wide) * stride;   // one packet per lane
  if (bf.pk_len < pk_need) {
    if (bf.pk) cudaFree(bf.pk);
    bf.pk = nullptr;
    bf.pk_len = 0;
    if (cudaMalloc(&bf.pk, pk_need * sizeof(double)) != cudaSuccess)
      return bail(fail(DDNM_ENOMEM, "cannot allocate the evaluation packets"));
    bf.pk_len = pk_need;
  }
  d->wide_pk_cap = bf.pk_len;
  const int32_t bounds[2] = {0, c->nb};
  int check = 4;
  if (const char* e = getenv("DDNM_DD_CHECK")) check = std::max(1, atoi(e));
  int32_t active = B;
  c->last_rounds = 0;
  c->last_launches = 2;               // init step, boundary values
  for (long long round = 0;; ++round) {
    if ((rc = ddnm_dd_eval(d, bf.pk, stride, s))) return bail(rc);
    const bool count = round % check == check - 1;
    if ((rc = ddnm_dd_step(d, bf.pk, 1, bounds, stride, s, count ? &active : nullptr))) return bail(rc);
    c->last_rounds += 1;
    c->last_launches += 5;            // compact, decoder, rows, pack, step
    if (count && active == 0) break;
    if (count) bf.wide.lane_bound = std::min<long long>(bf.wide.vpad, (long long)active * 16);
  }
  bf.wide.lane_bound = 0;
  unsigned long long lanes = 0;
  if (cudaMemcpyAsync(&lanes, bf.wide.lanes_total, sizeof lanes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return bail(fail(DDNM_ECUDA, "cannot read the lane count"));
  c->last_lanes = (long long)lanes;
  return ddnm_dd_end(d);
}

