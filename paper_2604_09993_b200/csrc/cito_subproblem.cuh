// cito_subproblem.cuh — device assembly of the SCP subproblem's CSC matrices
// (SURVEY.md §8(f) row 1): replaces cito.scp.build_subproblem's row loops and
// cito.conic.canonicalize/_to_csc (/root/reference/pkg/src/cito/scp.py:160-351,
// conic.py:99-125, 209-269).
//
// The host lays out a superset CSC (every entry that can be nonzero, rows
// sorted inside each column) with a recipe per entry: a constant, or
// (sign * LIN[src][idx]) * sigma[col] for the linearized rows.  Per iteration:
//   k_csc_count   warp per column: evaluate, count exact nonzeros
//   k_scan        single CTA: exclusive scan of the counts -> indptr (int32)
//   k_csc_write   warp per column: evaluate again, ballot-compact the nonzeros
// which is the reference's `keep = vals != 0` + eliminate_zeros + sort_indices.
// k_rhs forms b / h of the linearized rows (warp per row, up to 3 segments).
#pragma once

#include <cstdint>

struct LinTable {
  const double* p[10];  // jx, ju, js, imp_jac, theta_jac, psi_jac, ends, imp_v, theta, psi
};

__device__ __forceinline__ double sp_value(int64_t e, double sig, const int8_t* __restrict__ src,
                                           const int64_t* __restrict__ idx, const double* __restrict__ val,
                                           const LinTable& L) {
  const int s = src[e];
  return s < 0 ? val[e] : (val[e] * L.p[s][idx[e]]) * sig;
}

__global__ void __launch_bounds__(256) k_csc_count(int32_t ncols, const int64_t* __restrict__ sp_ptr,
                                                   const int8_t* __restrict__ src, const int64_t* __restrict__ idx,
                                                   const double* __restrict__ val, const double* __restrict__ sigma,
                                                   const LinTable L, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const double sig = sigma[c];
  int n = 0;
  for (int64_t e = sp_ptr[c] + lane; e < sp_ptr[c + 1]; e += 32) n += sp_value(e, sig, src, idx, val, L) != 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (lane == 0) counts[c] = n;
}

__global__ void __launch_bounds__(1024) k_scan(int32_t n, const int32_t* __restrict__ counts,
                                               int32_t* __restrict__ out_ptr) {
  __shared__ int32_t part[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < n; base += 1024) {
    const int32_t i = base + threadIdx.x;
    int32_t v = i < n ? counts[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
      const int32_t t = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) out_ptr[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) out_ptr[n] = carry;
}

__global__ void __launch_bounds__(256) k_csc_write(int32_t ncols, const int64_t* __restrict__ sp_ptr,
                                                   const int32_t* __restrict__ row, const int8_t* __restrict__ src,
                                                   const int64_t* __restrict__ idx, const double* __restrict__ val,
                                                   const double* __restrict__ sigma, const LinTable L,
                                                   const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_rows,
                                                   double* __restrict__ out_vals) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const double sig = sigma[c];
  int32_t base = out_ptr[c];
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t e0 = sp_ptr[c]; e0 < sp_ptr[c + 1]; e0 += 32) {
    const int64_t e = e0 + lane;
    const bool in = e < sp_ptr[c + 1];
    const double v = in ? sp_value(e, sig, src, idx, val, L) : 0.0;
    const bool nz = in && v != 0.0;
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (nz) {
      const int32_t pos = base + __popc(m & lt);
      out_rows[pos] = row[e];
      out_vals[pos] = v;
    }
    base += __popc(m);
  }
}

__global__ void __launch_bounds__(256) k_rhs(int64_t nrows, const int32_t* __restrict__ rows,
                                             const int8_t* __restrict__ form, const int8_t* __restrict__ vsrc,
                                             const int64_t* __restrict__ voff, const int8_t* __restrict__ seg_src,
                                             const int64_t* __restrict__ seg_off, const int32_t* __restrict__ seg_len,
                                             const int64_t* __restrict__ seg_cb, const int64_t* __restrict__ cols,
                                             const double* __restrict__ z, const LinTable L,
                                             double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= nrows) return;
  double dot = 0.0;
#pragma unroll
  for (int sgi = 0; sgi < 3; ++sgi) {
    const int s = seg_src[3 * i + sgi];
    if (s < 0) continue;
    const double* J = L.p[s] + seg_off[3 * i + sgi];
    const int64_t* cz = cols + seg_cb[3 * i + sgi];
    const int len = seg_len[3 * i + sgi];
    for (int j = lane; j < len; j += 32) dot += J[j] * z[cz[j]];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) {
    const double v = L.p[vsrc[i]][voff[i]];
    out[rows[i]] = form[i] == 0 ? v - dot : dot - v;  // dynamics: ends - J.ref ; others: J.ref - value
  }
}
