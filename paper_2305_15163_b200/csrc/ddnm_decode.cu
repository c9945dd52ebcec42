// Batched full decode of the SQP solutions: RomInstance.decode
// (driver.py:148-152) -- per block the full interior map and the interface
// map applied to their latent slices -- and, given restricted FOM states,
// relative_error (driver.py:496-507).
//
// Grid: x = mu tiles of `mu_tile` (<= DEC_MU) parameters, y = decoder jobs.
// A CTA stages its tile's latents in shared memory, computes the hidden
// activations of its decoder for the whole tile (shared, [mu][hidden]) and
// then sweeps the output rows with one thread per row, reading W2 in the
// ELL-transposed layout (consecutive threads = consecutive rows = coalesced)
// once for the whole tile.  The arithmetic follows the reference's operation
// order without contraction: z = b1 + sum_d W1[:, d] x_d (autoencoder.py:
// 134-140), raw = sum over the CSR row in storage order (scipy csr_matvec),
// raw * scale + shift (autoencoder.py:147).
#include "ddnm_device.cuh"

namespace ddnm {

cudaError_t raise_smem_limit(const void* fn, size_t bytes);   // ddnm_abi.cu


constexpr int DEC_MU = 8;
constexpr int DEC_THREADS = 256;

__device__ __forceinline__ double act_only(int act, double z, const double* tab) {
  // per map: interior swish, SRPC port nets sigmoid
  const double s = expit_fast(z, tab);
  return act == ACT_SWISH ? __dmul_rn(z, s) : s;   // autoencoder.py:31-36
}

__global__ void __launch_bounds__(DEC_THREADS) k_decode(DecodeParams p) {
  extern __shared__ double dsm[];
  const DecodeJob& J = p.jobs[blockIdx.y];
  const DecDev& D = J.D;
  const int MU = p.mu_tile;
  const int mu0 = blockIdx.x * MU;
  const int nmu = min(MU, p.B - mu0);
  const int lat = J.lat;
  double* xs = dsm;                        // [DEC_MU][32]
  double* hid = dsm + DEC_MU * 32;         // [MU][n_hidden]
  __shared__ double red[DEC_THREADS / 32][DEC_MU][2];
  for (int i = threadIdx.x; i < DEC_MU * 32; i += blockDim.x) {
    const int m = i >> 5, d = i & 31;
    xs[i] = (m < nmu && d < lat) ? p.x[(size_t)(mu0 + m) * p.n_D + J.x_off + d] : 0.0;
  }
  __syncthreads();
  const int H = D.n_hidden;
  if (!p.linear) {
    for (int k = threadIdx.x; k < H; k += blockDim.x) {
      double z[DEC_MU];
      const double b = __ldg(D.b1 + k);
#pragma unroll
      for (int m = 0; m < DEC_MU; ++m) z[m] = b;
      for (int d = 0; d < lat; ++d) {
        const double w = __ldg(D.W1t + (size_t)d * D.ldw + k);
#pragma unroll
        for (int m = 0; m < DEC_MU; ++m) z[m] = __dadd_rn(z[m], __dmul_rn(w, xs[m * 32 + d]));
      }
#pragma unroll
      for (int m = 0; m < DEC_MU; ++m)
        if (m < MU) hid[(size_t)m * H + k] = act_only(D.act, z[m], k_exp2_32);
    }
    __syncthreads();
  }
  double num[DEC_MU], den[DEC_MU];
#pragma unroll
  for (int m = 0; m < DEC_MU; ++m) num[m] = den[m] = 0.0;
  const int n_out = D.n_out;
  for (int o = threadIdx.x; o < n_out; o += blockDim.x) {
    double acc[DEC_MU];
#pragma unroll
    for (int m = 0; m < DEC_MU; ++m) acc[m] = 0.0;
    if (!p.linear) {
      const int w = __ldg(D.indptr + o + 1) - __ldg(D.indptr + o);
      const int k0 = D.ell_k0 ? __ldg(D.ell_k0 + o) : 0;
      for (int e = 0; e < w; ++e) {
        const double v = __ldg(D.ell_v + (size_t)e * n_out + o);
        const int k = D.ell_k0 ? k0 + e : __ldg(D.ell_k + (size_t)e * n_out + o);
#pragma unroll
        for (int m = 0; m < DEC_MU; ++m)
          if (m < MU) acc[m] = __dadd_rn(acc[m], __dmul_rn(v, hid[(size_t)m * H + k]));
      }
      const double scl = __ldg(D.scale + o), sh = __ldg(D.shift + o);
#pragma unroll
      for (int m = 0; m < DEC_MU; ++m) acc[m] = __dadd_rn(__dmul_rn(acc[m], scl), sh);
    } else {
      for (int d = 0; d < lat; ++d) {
        const double v = __ldg(D.W1 + (size_t)o * lat + d);
#pragma unroll
        for (int m = 0; m < DEC_MU; ++m) acc[m] = __dadd_rn(acc[m], __dmul_rn(v, xs[m * 32 + d]));
      }
    }
#pragma unroll
    for (int m = 0; m < DEC_MU; ++m) {
      if (m >= nmu) continue;
      const size_t at = (size_t)(mu0 + m) * p.state_len + J.out_off + o;
      if (p.states) p.states[at] = acc[m];
      if (p.fom) {
        const double f = p.fom[at];
        const double r = f - acc[m];
        num[m] = fma(r, r, num[m]);
        den[m] = fma(f, f, den[m]);
      }
    }
  }
  if (!p.fom) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < DEC_MU; ++m) {
    const double a = warp_sum(num[m]), b = warp_sum(den[m]);
    if (lane == 0) { red[wid][m][0] = a; red[wid][m][1] = b; }
  }
  __syncthreads();
  if (threadIdx.x < 2 * nmu) {
    const int m = threadIdx.x >> 1, q = threadIdx.x & 1;
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][m][q];
    p.part[((size_t)(mu0 + m) * p.n_jobs + blockIdx.y) * 2 + q] = t;
  }
}

// relative_error (driver.py:496-507) per mu from the per-job partial sums;
// NaN for a zero-norm reference block (the reference raises ValueError).
__global__ void k_decode_err(DecodeParams p) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p.B) return;
  const double* q = p.part + (size_t)k * p.n_jobs * 2;
  double total = 0.0;
  bool zero = false;
  for (int b = 0; b < p.nb; ++b) {
    const double num = q[4 * b] + q[4 * b + 2];
    const double den = q[4 * b + 1] + q[4 * b + 3];
    if (den == 0.0) zero = true;
    total += num / den;
  }
  p.err[k] = zero ? NAN : sqrt(total / p.nb);
}

// smem bytes of k_decode for a tile of `mu` parameters
size_t decode_smem(int mu, int max_hidden) {
  return ((size_t)DEC_MU * 32 + (size_t)mu * max_hidden) * sizeof(double);
}

int decode_mu_tile(int max_hidden, size_t smem_cap) {
  for (int mu = DEC_MU; mu >= 1; mu >>= 1)
    if (decode_smem(mu, max_hidden) <= smem_cap) return mu;
  return 0;
}

cudaError_t launch_decode(const DecodeParams& p, cudaStream_t s) {
  if (p.B == 0) return cudaSuccess;
  const size_t smem = decode_smem(p.linear ? 0 : p.mu_tile, p.max_hidden);
  cudaError_t e = raise_smem_limit((const void*)k_decode, smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((p.B + p.mu_tile - 1) / p.mu_tile, p.n_jobs);
  k_decode<<<grid, DEC_THREADS, smem, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p.fom) {
    k_decode_err<<<(p.B + 127) / 128, 128, 0, s>>>(p);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ddnm
